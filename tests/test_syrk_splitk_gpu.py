"""Split-K curvature SYRK (umma_gemm.cuh split_k_epilogue, kfac_ops.cu
bf16_k_split): a launch of few 128x128 tiles splits every tile's k-blocks over
a cluster of 2 or 4 CTAs (8 when forced) and sums the partial tiles over distributed shared
memory in cluster-rank order.

Checks: the split factors match an fp64 product of the same bf16 inputs to
fp32 accumulation (<= 1e-5 relative Frobenius, the SYRK bar of
test_kfac_gpu.py); the result is the same bits on every call (the reduction
order does not depend on which CTA finishes first); accumulate (beta = 1),
the mirrored upper triangle, ragged d / n, token-major operands and grouped
launches go through the split epilogue; forced factors (PF_KSPLIT, read once
per process, so in a subprocess) including slices with no k-blocks."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def K():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2211_14133_b200 import kfac
    assert kfac.device_ok(), "libpf_b200.so needs an sm_100 device"
    return kfac


def tape(seed, d, n, token_major=False):
    g = torch.Generator(device="cuda").manual_seed(seed)
    if token_major:
        return torch.randn((n, (d + 7) // 8 * 8), generator=g, device="cuda").to(torch.bfloat16)[:, :d]
    return torch.randn((d, (n + 7) // 8 * 8), generator=g, device="cuda").to(torch.bfloat16)[:, :n]


def want_of(x, scale, token_major=False, base=None):
    xd = x.double()
    w = scale * (xd.t() @ xd if token_major else xd @ xd.t())
    return w if base is None else w + base.double()


def rel(got, want):
    return float((got.double() - want).norm() / want.norm())


# d, n: 36 tiles x 64 k-blocks -> 2 slices; 6 tiles -> 4; 21 tiles x 16 -> 2;
# ragged d (partial tile) and n (partial last k-block, short last slice)
@pytest.mark.parametrize("d,n", [(1024, 4096), (384, 4096), (768, 1024), (200, 4136), (2048, 4096), (256, 2048)])
def test_split_syrk_matches_fp64_and_is_deterministic(K, d, n):
    x = tape(d + n, d, n)
    if n % 8:
        x = K.to_tape_layout(x)
    f1 = torch.empty((d, d), device="cuda")
    f2 = torch.empty((d, d), device="cuda")
    K.syrk([(x, f1, 1.0 / n, False)], fill_upper=True)
    K.syrk([(x, f2, 1.0 / n, False)], fill_upper=True)
    torch.cuda.synchronize()
    assert torch.equal(f1, f2)
    assert torch.equal(f1, f1.t())
    assert rel(f1, want_of(x[:, :n], 1.0 / n)) <= 1e-5


def test_split_syrk_accumulate_lower_only_token_major_grouped(K):
    xa = tape(1, 1024, 4096, token_major=True)
    xb = tape(2, 512, 4096, token_major=True)
    fa = torch.full((1024, 1024), 0.25, device="cuda")
    fb = torch.full((512, 512), -1.0, device="cuda")
    fa0, fb0 = fa.clone(), fb.clone()
    K.syrk([(xa, fa, 0.5, True, True), (xb, fb, 2.0, True, True)], fill_upper=False)
    torch.cuda.synchronize()
    il = torch.tril_indices(1024, 1024, device="cuda")
    wa = want_of(xa, 0.5, True, fa0)
    assert rel(fa[il[0], il[1]], wa[il[0], il[1]]) <= 1e-5
    r = torch.arange(1024, device="cuda") // 128
    above = r[None, :] > r[:, None]  # tiles right of the diagonal tile: never written
    assert torch.equal(fa[above], fa0[above])
    il = torch.tril_indices(512, 512, device="cuda")
    wb = want_of(xb, 2.0, True, fb0)
    assert rel(fb[il[0], il[1]], wb[il[0], il[1]]) <= 1e-5


SNIPPET = r"""
import json, sys, torch
sys.path.insert(0, %r)
from paper_2211_14133_b200 import kfac as K
out = {}
for d, n in ((384, 4096), (300, 576), (128, 64)):
    g = torch.Generator(device="cuda").manual_seed(d + n)
    x = torch.randn((d, n), generator=g, device="cuda").to(torch.bfloat16)
    f = torch.full((d, d), 3.0, device="cuda")
    K.syrk([(x, f, 1.0 / n, True)], fill_upper=True)
    torch.cuda.synchronize()
    xd = x.double()
    w = 3.0 + (xd @ xd.t()) / n
    out["%%d_%%d" %% (d, n)] = float((f.double() - w).norm() / w.norm())
    out["sym_%%d_%%d" %% (d, n)] = bool(torch.equal(f, f.t()))
print(json.dumps(out))
""" % ROOT


@pytest.mark.parametrize("ks", ["1", "2", "4", "8"])
def test_forced_split_factors(ks):
    """PF_KSPLIT forces the factor for every bf16 launch: 576 tokens = 9
    k-blocks over 8 slices leaves slices with no k-blocks (their partial is
    zero), 64 tokens = one k-block for all of them."""
    env = dict(os.environ, PF_KSPLIT=ks)
    out = subprocess.run([sys.executable, "-c", SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    for k, v in res.items():
        if k.startswith("sym_"):
            assert v, k
        else:
            assert v <= 1e-5, (k, v)


WIDE_SNIPPET = r"""
import json, sys, torch
sys.path.insert(0, %r)
from paper_2211_14133_b200 import kfac as K
out = {}
cases = ((384, 512, False, True), (200, 136, False, True), (640, 1024, True, True), (1024, 4096, True, False),
         (4096, 512, False, True))
for d, n, tm, fill in cases:
    g = torch.Generator(device="cuda").manual_seed(d + n)
    x = torch.randn((n, d) if tm else (d, n), generator=g, device="cuda").to(torch.bfloat16)
    f = torch.full((d, d), 0.5, device="cuda")
    K.syrk([(x, f, 1.0 / n, True, tm)], fill_upper=fill)
    torch.cuda.synchronize()
    xd = x.double()
    w = 0.5 + ((xd.t() @ xd) if tm else (xd @ xd.t())) / n
    key = "%%d_%%d_%%d_%%d" %% (d, n, tm, fill)
    blk = torch.arange(d, device="cuda") // 128
    low = blk[None, :] <= blk[:, None]  # 128-blocks on or left of the diagonal block
    out[key] = float((f.double() - w)[low].norm() / w[low].norm())
    if fill:
        out["sym_" + key] = bool(torch.equal(f, f.t())) and float((f.double() - w).norm() / w.norm()) <= 1e-5
    else:
        out["sym_" + key] = bool(torch.equal(f[~low], torch.full_like(f[~low], 0.5)))  # never written
print(json.dumps(out))
""" % ROOT


@pytest.mark.parametrize("wide", ["0", "2"])
def test_wide_tiles_forced(wide):
    """PF_SYRK_WIDE=2 runs every SYRK on 128 x 256 tiles (default: launches of
    more 128-wide tiles than SMs): ragged d with a 256-wide tile whose second
    128-row B box lies wholly past d (d = 384), partial tiles (d = 200),
    token-major operands, accumulate, lower-only (blocks right of the diagonal
    block never written) and the mirrored upper triangle."""
    env = dict(os.environ, PF_SYRK_WIDE=wide)
    out = subprocess.run([sys.executable, "-c", WIDE_SNIPPET], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    for k, v in res.items():
        if k.startswith("sym_"):
            assert v, k
        else:
            assert v <= 1e-5, (k, v)
