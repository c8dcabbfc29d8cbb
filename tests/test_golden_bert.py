"""CPU pinning of the BERT-shaped reference goldens (tests/golden/kfac_bert.npz):
the sketches the compiled reference produced are checked against an
independent numpy FP64 computation on the regenerated inputs, so the GPU
parity tests (test_bert_golden_gpu.py) compare against numbers that are
known to be right.  ~10 s on 8 cores."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import make_bert_golden as G  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "kfac_bert.npz")


@pytest.fixture(scope="module")
def gold():
    return dict(np.load(GOLDEN))


_factors = {}


def factor(d):
    if d not in _factors:
        a = G.tape(d)
        _factors[d] = (a, (a @ a.T) / G.N_TOKENS)
    return _factors[d]


@pytest.mark.parametrize("d", G.SIZES)
def test_golden_factor_and_tape(gold, d):
    a, A = factor(d)
    assert G.tape_sha(a) == str(gold[f"d{d}_tape_sha"])
    sk = A @ G.omega(d)
    want = gold[f"d{d}_factor_sk"]
    assert np.linalg.norm(sk - want) / np.linalg.norm(want) < 1e-13  # FP64 vs FP64, order only
    assert np.allclose(A[G.SAMPLE_ROWS(d)], gold[f"d{d}_factor_rows"], rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("lam", G.LAMBDAS)
@pytest.mark.parametrize("d", G.SIZES)
def test_golden_inverse_solves_the_damped_factor(gold, d, lam):
    """(fp32(A) + lambda I) (A^-1 Omega) = Omega to FP64 accuracy x kappa."""
    _, A = factor(d)
    a32 = A.astype(np.float32).astype(np.float64) + lam * np.eye(d)
    sk = gold[f"d{d}_inv_{lam:g}_sk"]
    err = np.abs(a32 @ sk - G.omega(d)).max()
    assert err < 1e-9, err


@pytest.mark.parametrize("shape", G.PREC)
def test_golden_precondition_consistent(gold, shape):
    """The reference's P = B^-1 G A^-1 on the sampled rows equals
    (B^-1)[rows] G A^-1 with both inverses recomputed by numpy (LU, FP64)
    from the same fp32 factors."""
    d_out, d_in = shape
    _, A = factor(d_in)
    _, B = factor(d_out)
    ai = np.linalg.inv(A.astype(np.float32).astype(np.float64) + 0.1 * np.eye(d_in))
    bi = np.linalg.inv(B.astype(np.float32).astype(np.float64) + 0.1 * np.eye(d_out))
    P_rows = bi[G.SAMPLE_ROWS(d_out)] @ G.gradient(d_out, d_in) @ ai
    want = gold[f"p{d_out}x{d_in}_rows"].astype(np.float64)
    assert np.linalg.norm(P_rows - want) / np.linalg.norm(want) < 1e-6
