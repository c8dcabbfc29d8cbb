"""The A/B switches of the inversion and GEMM launch policies
change only scheduling -- tile widths, launch priorities, persistent tiles,
side-stream placement, group start times, slicing kernels -- never the
arithmetic: every switch must give bit-identical inverses, digit forms and
preconditioned weights.  Each configuration runs in a fresh process (the
switches are read once per process)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SNIPPET = r"""
import hashlib, json, sys, torch
sys.path.insert(0, %r)
from paper_2211_14133_b200 import kfac as K
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(7)
mats = []
for d in (2048, 2048, 1024, 300):
    x = torch.randn(d, 2048, generator=g, device="cuda")
    mats.append(x @ x.T / 2048)
outs = [torch.empty_like(m) for m in mats]
digs = [torch.empty(K.slice_bytes(m.shape[0], m.shape[0]), dtype=torch.uint8, device="cuda") for m in mats]
K.damped_inverse_batched(mats, 0.1, outs, digs, check=True)
items = []
for a, b in ((2, 0), (0, 2)):  # (d_in, d_out) = (1024, 2048) and (2048, 1024)
    w = 0.02 * torch.randn(outs[b].shape[0], outs[a].shape[0], generator=g, device="cuda")
    gr = torch.randn(w.shape, generator=g, device="cuda")
    items.append((w, gr, K.SlicedMatrix(outs[a], digs[a]), K.SlicedMatrix(outs[b], digs[b]), 1e-3))
K.precondition_update_sliced(items)
torch.cuda.synchronize()
h = hashlib.sha256()
for t in outs + digs + [it[0] for it in items]:
    h.update(t.cpu().numpy().tobytes())
print(json.dumps({"sha": h.hexdigest()}))
""" % ROOT

SWITCHES = ["PF_NO_NSPLIT=1", "PF_NO_PRIO=1", "PF_GEMM_PERSIST=0", "PF_EARLY_TRTRI=0", "PF_EARLY_ROOT=0", "PF_INV_DELAY=0",
            "PF_SLICE_SHORT=0", "PF_WARP_SLICE_2K=0", "PF_NO_PDL=1", "PF_TRTRI_SPINE=0", "PF_READY_FLAGS=0",
            "PF_INV_GROUP_LEAD=0"]


def run(env_kv=None):
    env = dict(os.environ)
    for k in [s.split("=")[0] for s in SWITCHES]:
        env.pop(k, None)
    if env_kv:
        k, v = env_kv.split("=")
        env[k] = v
    out = subprocess.run([sys.executable, "-c", SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])["sha"]


@pytest.fixture(scope="module")
def baseline():
    return run()


@pytest.mark.parametrize("switch", SWITCHES)
def test_switch_is_bit_identical(baseline, switch):
    assert run(switch) == baseline
