"""The right-looking chain's fp32 diagonal update (diag_update_kernel,
PF_DIAG_FP32) against the digit-GEMM update it replaces: both
within the inverse residual bound, agreeing to rounding, at ragged sizes
(n < 128 tail blocks) forced onto the fp32 path with PF_DIAG_FP32_MIN_D=0,
and independent of what else is in the call.  Fresh processes: the switches
are read once per process."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DIMS = (130, 300, 520, 1000, 2048)

SNIPPET = r"""
import json, sys, torch
sys.path.insert(0, %r)
from paper_2211_14133_b200 import kfac as K
torch.cuda.set_device(0)
dims = %r
mats = []
for i, d in enumerate(dims):
    g = torch.Generator(device="cuda").manual_seed(100 + i)
    x = torch.randn(d, 1024, generator=g, device="cuda")
    mats.append(x @ x.T / 1024)
res = {}
batch = K.damped_inverse_batched(mats, 0.1)
alone = [K.damped_inverse_batched([m], 0.1)[0] for m in mats]
for d, m, inv, a in zip(dims, mats, batch, alone):
    A = (m + 0.1 * torch.eye(d, device="cuda")).double()
    r = (A @ inv.double() - torch.eye(d, device="cuda", dtype=torch.float64)).abs().max().item()
    res[str(d)] = {"residual": r, "same_alone": bool(torch.equal(inv, a)), "inv": inv.double().cpu().flatten()[::97].tolist()}
print(json.dumps(res))
""" % (ROOT, DIMS)


def run(env_extra):
    env = dict(os.environ)
    for k in ("PF_DIAG_FP32", "PF_DIAG_FP32_MIN_D", "PF_INV_GROUP_LEAD"):
        env.pop(k, None)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_fp32_diag_update_matches_digit_update():
    fp32 = run({"PF_DIAG_FP32_MIN_D": "0"})
    digit = run({"PF_DIAG_FP32": "0"})
    for d in map(str, DIMS):
        assert fp32[d]["residual"] <= 1e-5 and digit[d]["residual"] <= 1e-5, (d, fp32[d], digit[d])
        # a factor's bits never depend on the rest of the call
        assert fp32[d]["same_alone"] and digit[d]["same_alone"], d
        a, b = fp32[d]["inv"], digit[d]["inv"]
        scale = max(abs(v) for v in b)
        assert max(abs(x - y) for x, y in zip(a, b)) <= 1e-5 * scale, d
