"""Digit form (pf_slice) against its definition, bit for bit.

The fp32-accurate tensor-core GEMMs consume every fp32 operand row as
    x = 2^e (q0 2^-7 + q1 2^-14 + q2 2^-21 + q3 2^-28),  q_s in [-127, 127],
e = frexp exponent of max|row| (0 for an all-zero row), digits by successive
truncation of t = x 2^(7-e) in exact fp32 steps and a round-to-nearest-even
last digit clamped to +-127 (slice.cuh header).  The restatement below is
that definition in numpy; the kernels (warp per row, block per row, the
two-pass long-row path, the unaligned scalar path) use integer and packed
byte arithmetic instead, so this pins them to it.  Row norms (fp64, of the
represented row scaled by 2^-e) to 1e-15 relative.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2211_14133_b200 import kfac
    assert kfac.device_ok(), "libpf_b200.so needs an sm_100 device"
    return kfac


def digits_ref(x):
    """numpy restatement: (planes [4, rows, k] int8, exps [rows], sqnorm [rows])."""
    x = np.asarray(x, np.float32)
    rows, k = x.shape
    m = np.abs(x).max(axis=1)
    e = np.where(m > 0, np.frexp(m)[1], 0).astype(np.int32)
    t = (x.astype(np.float64) * np.exp2(7.0 - e)[:, None]).astype(np.float32)  # exact scaling
    q = []
    for _ in range(3):
        d = np.trunc(t)
        q.append(d)
        t = ((t - d) * np.float32(128)).astype(np.float32)
    q.append(np.clip(np.rint(t), -127, 127))
    planes = np.stack(q).astype(np.int8)
    qi = planes.astype(np.int64)
    big_q = ((qi[0] * 128 + qi[1]) * 128 + qi[2]) * 128 + qi[3]
    sq = np.array([float(sum(int(v) * int(v) for v in row)) * 2.0 ** -56 for row in big_q])
    return planes, e, sq


def unpack(K, buf, rows, k):
    kpad = (k + 15) // 16 * 16
    plane = (rows * kpad + 255) // 256 * 256
    b = buf.cpu().numpy()
    planes = np.stack([b[p * plane: p * plane + rows * kpad].view(np.int8).reshape(rows, kpad)[:, :k]
                       for p in range(4)])
    off = 4 * plane
    exps = b[off: off + 4 * rows].view(np.int32)
    off += (4 * rows + 255) // 256 * 256
    sq = b[off: off + 8 * rows].view(np.float64)
    return planes, exps, sq


CASES = [
    (64, 101, "normal"),      # rows not 16-byte aligned: scalar warp path
    (200, 128, "normal"),     # 8 lanes per row (rows <= 256)
    (96, 256, "scaled"),      # 8 lanes per row, zero rows and sign flips
    (40, 36, "normal"),       # 8 lanes per row, rows shorter than the group
    (300, 1024, "normal"),    # warp path, single pass
    (257, 1500, "scaled"),    # block-per-row path, zero rows, sign flips, huge/tiny row scales
    (96, 4096, "normal"),     # block-per-row path
    (40, 8192, "scaled"),     # block-per-row path at its maximum
    (24, 9000, "normal"),     # two-pass warp path (rows > 8192)
    (33, 2048, "ties"),       # last digit exactly half-way: ties to even
    (16, 512, "subnormal"),   # rows of subnormal values
]


@pytest.mark.parametrize("rows,k,kind", CASES)
def test_slice_matches_definition(K, rows, k, kind):
    g = torch.Generator().manual_seed(rows * 7 + k)
    x = torch.randn(rows, k, generator=g)
    if kind == "scaled":
        x = x * torch.exp(torch.randn(rows, 1, generator=g) * 20)
        x[::7] = 0
        x[3, ::3] = -x[3, ::3]
    elif kind == "ties":  # |x| 2^(28-e) = q + 1/2 exactly (<= 24 significant bits), e fixed by x[:, 0]
        q = torch.randint(0, 1 << 22, (rows, k), generator=g).double() + 0.5
        sgn = torch.where(torch.rand(rows, k, generator=g) < 0.5, -1.0, 1.0).double()
        x = (sgn * q * 2.0 ** -28).float()
        x[:, 0] = 0.75
    elif kind == "subnormal":
        x = x * 1e-39
    buf = torch.zeros(K.slice_bytes(rows, k), dtype=torch.uint8, device="cuda")
    xd = x.cuda()
    from paper_2211_14133_b200 import _lib as L
    L.check(L.lib().pf_slice(xd.data_ptr(), rows, k, k, buf.data_ptr(), K._stream()), "slice")
    torch.cuda.synchronize()
    planes, exps, sq = unpack(K, buf, rows, k)
    p_ref, e_ref, sq_ref = digits_ref(x.numpy())
    assert np.array_equal(exps, e_ref)
    assert np.array_equal(planes, p_ref), f"{(planes != p_ref).sum()} digit bytes differ"
    np.testing.assert_allclose(sq, sq_ref, rtol=1e-15, atol=0)
