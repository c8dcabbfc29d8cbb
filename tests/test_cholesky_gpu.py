"""GPU cholesky_factor (pf_cholesky_factor through the C-ABI) against the
oracle -- reference proj/src/kfac/matrix.cpp:117-134.

Tolerances: L relative Frobenius <= 1e-5 vs the FP64 oracle factor of the
same fp32 matrix (fp32-accurate factorisation: measured ~1e-7); the strictly
upper triangle exactly zero; ||L L^T - M|| / ||M|| <= 1e-6 at every size,
including the BERT-Large d = 4096 (fp64 check on the device).  Pivot failures
report the reference's 1-based column (matrix.cpp:124-125)."""
import numpy as np
import pytest
import torch

from oracle import ref as R

pytestmark = pytest.mark.gpu

L_TOL = 1e-5
RECON_TOL = 1e-6


@pytest.fixture(scope="module")
def K():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2211_14133_b200 import kfac
    assert kfac.device_ok(), "libpf_b200.so needs an sm_100 device"
    return kfac


def spd32(seed, d, n=None):
    n = n or max(2 * d, 64)
    x = R.orc_symmetric(seed, (d, n), 3 ** 0.5)
    m = (x @ x.T) / n
    return m.astype(np.float32)


def rel_fro(got, want):
    return float(np.linalg.norm(np.asarray(got, np.float64) - want) / np.linalg.norm(want))


@pytest.mark.parametrize("d", [1, 5, 37, 128, 129, 300, 640, 1024])
def test_cholesky_factor_matches_oracle(K, d):
    m = spd32(700 + d, d)
    got = K.cholesky_factor(torch.from_numpy(m).cuda()).cpu().numpy()
    want = R.orc_cholesky_factor(m.astype(np.float64))
    assert np.all(np.triu(got, 1) == 0.0)
    assert np.all(np.diag(got) > 0)
    assert rel_fro(got, want) <= L_TOL
    g64 = got.astype(np.float64)
    assert rel_fro(g64 @ g64.T, m.astype(np.float64)) <= RECON_TOL


def test_cholesky_factor_damping_and_strided_input(K):
    d, lam = 300, 0.25
    big = torch.zeros((d, d + 12), dtype=torch.float32, device="cuda")
    m = spd32(11, d)
    big[:, :d] = torch.from_numpy(m)
    got = K.cholesky_factor(big[:, :d], damping=lam).cpu().numpy().astype(np.float64)
    want = m.astype(np.float64) + lam * np.eye(d)
    assert rel_fro(got, R.orc_cholesky_factor(want)) <= L_TOL
    assert rel_fro(got @ got.T, want) <= RECON_TOL


@pytest.mark.parametrize("d", [2048, 4096])
def test_cholesky_factor_bert_shapes(K, d):
    x = torch.from_numpy(R.orc_symmetric(d, (d, 4096), 3 ** 0.5)).to(torch.bfloat16).cuda().float()
    m = (x @ x.T) / 4096 + 0.1 * torch.eye(d, device="cuda")
    lo = K.cholesky_factor(m).double()
    assert torch.count_nonzero(torch.triu(lo, 1)).item() == 0
    rec = torch.linalg.norm(lo @ lo.T - m.double()) / torch.linalg.norm(m.double())
    assert rec.item() <= RECON_TOL
    # the factorisation is the one the damped inverse uses: X = L^-1 consistent
    ref = torch.linalg.cholesky(m.double())
    assert (torch.linalg.norm(lo - ref) / torch.linalg.norm(ref)).item() <= L_TOL


@pytest.mark.parametrize("d,col", [(2, 2), (37, 20), (300, 201), (1024, 900)])
def test_cholesky_factor_not_pd_reports_column(K, d, col):
    m = np.eye(d, dtype=np.float32)
    m[col - 1, col - 1] = -1.0
    with pytest.raises(K.NotPositiveDefinite) as e:
        K.cholesky_factor(torch.from_numpy(m).cuda())
    assert e.value.column == col
    with pytest.raises(R.DomainError):  # the reference raises too
        R.orc_cholesky_factor(m.astype(np.float64))


def test_cholesky_factor_nan_rejected(K):
    m = np.eye(64, dtype=np.float32)
    m[10, 10] = np.nan
    with pytest.raises(K.NotPositiveDefinite):
        K.cholesky_factor(torch.from_numpy(m).cuda())
