"""Pins the oracle before it is trusted (CPU only).

1. The compiled reference (oracle/_ref) reproduces the reference's own golden
   vectors: the frozen hex-float loss trajectories of proj/tests/test_kfac.cpp:
   430-446 and the hand cases of :99-169.
2. The C restatement (oracle/kfac_oracle.c) is BIT-IDENTICAL to the compiled
   reference on seeded inputs (same loop and operation order, FP64).
3. The pure-Python scheduler restatement (oracle/schedule_oracle.py) agrees
   with the compiled reference on every seeded table of the reference suites.
4. Committed numeric goldens (tests/golden/kfac_small.npz) match both.
"""
import os

import numpy as np
import pytest

from oracle import ref as R
from oracle import schedule_oracle as O

import helpers as H

need_ref = pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")
GOLD = os.path.join(os.path.dirname(__file__), "golden", "kfac_small.npz")


@need_ref
def test_reference_reproduces_frozen_loss_trajectories():
    k = R.ref_train_toy(steps=60, lr=1e-3, damping=1e-3, refresh=1, kfac=True)
    assert k[0] == float.fromhex("0x1.25c8e49540d51p-2")
    assert k[1] == float.fromhex("0x1.3721e259f68c2p-5")
    assert k[2] == float.fromhex("0x1.14b029c846e3dp-12")
    assert k[10] == float.fromhex("0x1.736e63d7c6afep-29")
    g = R.ref_train_toy(steps=60, lr=4.0, kfac=False)
    assert g[1] == float.fromhex("0x1.6a346e8f5a894p-4")
    assert g[22] == float.fromhex("0x1.00f354834db91p-10")


def test_oracle_hand_cases():
    """proj/tests/test_kfac.cpp:99-169 against the C restatement."""
    a = R.orc_curvature_factor(np.array([[1.0], [2.0]]))
    assert a.tolist() == [[1.0, 2.0], [2.0, 4.0]]
    assert R.orc_curvature_factor(np.array([[3.0]])).tolist() == [[9.0]]
    assert np.abs(R.orc_curvature_factor(np.array([[1.0, 1.0], [2.0, 2.0]])) - a).max() < 1e-15
    inv = R.orc_cholesky_spd_inverse(np.array([[4.0, 0.0], [0.0, 9.0]]), 0.0)
    assert np.abs(inv - np.array([[0.25, 0.0], [0.0, 1 / 9]])).max() < 1e-15
    assert np.abs(R.orc_cholesky_spd_inverse(np.eye(3), 0.0) - np.eye(3)).max() < 1e-15
    with pytest.raises(R.DomainError):
        R.orc_cholesky_spd_inverse(np.array([[1.0, 2.0], [2.0, 1.0]]), 0.0)
    p = R.orc_precondition(np.array([[6.0, 6.0]]), 0.5 * np.eye(2), np.array([[1 / 3]]))
    assert np.abs(p - np.array([[1.0, 1.0]])).max() < 1e-15


@need_ref
@pytest.mark.parametrize("d_in,d_out,n", [(3, 2, 5), (17, 9, 33), (64, 48, 100), (130, 70, 64)])
def test_c_restatement_bit_identical_to_reference(d_in, d_out, n):
    a = R.orc_symmetric(11 + d_in, (d_in, n), 3 ** 0.5)
    e = R.orc_symmetric(12 + d_out, (d_out, n), 3 ** 0.5)
    A, B = R.ref_curvature_factors(a, e)
    assert np.array_equal(R.orc_curvature_factor(a) * 1.0, A)
    assert np.array_equal(R.orc_curvature_factor(e), B)
    for lam in (0.1, 1e-3):
        Ai = R.ref_cholesky_spd_inverse(A, lam)
        assert np.array_equal(R.orc_cholesky_spd_inverse(A, lam), Ai)
    Ai = R.ref_cholesky_spd_inverse(A, 0.1)
    Bi = R.ref_cholesky_spd_inverse(B, 0.1)
    g = R.orc_symmetric(13, (d_out, d_in))
    assert np.array_equal(R.orc_precondition(g, Ai, Bi), R.ref_precondition(g, Ai, Bi))
    w = R.orc_symmetric(14, (d_out, d_in), 0.02)
    W_ref, plain = R.ref_ngd_step(w, g, Ai, Bi, 1e-3)
    assert not plain
    assert np.array_equal(R.orc_ngd_update(w, R.orc_precondition(g, Ai, Bi), 1e-3), W_ref)
    # missing inverses: plain gradient + flag (kfac.cpp:192-195)
    W_plain, plain = R.ref_ngd_step(w, g, None, None, 1e-3)
    assert plain and np.array_equal(W_plain, R.orc_ngd_update(w, g, 1e-3))


@need_ref
def test_splitmix_matches_reference():
    rng = H.SplitMix64(1618)
    mine = np.array([rng.symmetric() for _ in range(1000)])
    assert np.array_equal(mine, R.ref_splitmix(1618, 1000))
    assert np.array_equal(R.orc_symmetric(1618, (1000,)), mine)


def test_numeric_goldens():
    z = np.load(GOLD)
    for d_in, d_out, n in ((64, 32, 96), (130, 70, 200)):
        tag = f"{d_in}x{d_out}x{n}"
        a = R.orc_symmetric(1000 + d_in, (d_in, n), 3 ** 0.5)
        e = R.orc_symmetric(2000 + d_out, (d_out, n), 3 ** 0.5)
        A, B = R.orc_curvature_factor(a), R.orc_curvature_factor(e)
        assert np.array_equal(A, z[f"{tag}_A"]) and np.array_equal(B, z[f"{tag}_B"])
        Ai = R.orc_cholesky_spd_inverse(A, 0.1)
        assert np.array_equal(Ai, z[f"{tag}_Ainv"])
        Bi = R.orc_cholesky_spd_inverse(B, 0.1)
        g = R.orc_symmetric(3000 + d_in, (d_out, d_in), 1.0)
        assert np.array_equal(R.orc_precondition(g, Ai, Bi), z[f"{tag}_P"])


def _canon_ref(dump):
    return H.canonical(dump.items)


@need_ref
def test_python_schedule_oracle_matches_reference():
    rng = H.SplitMix64(1618)
    n_checked = 0
    for _ in range(200):
        cfg, costs, inv_par = H.acceptance_table(rng)
        want = R.ref_assign_dump(cfg, costs, inv_par, 10)
        try:
            got = O.assign_works(cfg, costs, inv_par, 10)
        except O.Infeasible as e:
            assert want.infeasible is not None
            assert e.deficit == want.infeasible[0]
            continue
        assert want.infeasible is None
        assert (got["period"], got["base_period"], got["refresh"], got["prior"]) == want.header[:4]
        mine = [it for line in got["lines"] for it in line]
        assert H.canonical(mine) == _canon_ref(want)
        assert got["staleness"] == want.staleness
        n_checked += 1
    assert n_checked >= 20
    for name, (cfg, costs) in H.bert_configs().items():
        want = R.ref_assign_dump(cfg, costs, True, 10)
        got = O.assign_works(cfg, costs, True, 10)
        assert H.canonical([it for line in got["lines"] for it in line]) == _canon_ref(want), name


@need_ref
@pytest.mark.parametrize("p2p", [0.0, 0.3, 1.0, 2.5])
def test_python_build_oracle_matches_reference(p2p):
    import paper_2211_14133_b200.schedule as S
    for method in (0, 1, 2):
        for depth in (2, 4, 6):
            cfg = H.make_config(method, depth, 2 * depth, 1, 2 if method == 2 else 1)
            t = S.CostTable(t_f=0.9, t_b=1.7, p2p_latency=p2p)
            lines, _ = O.build_schedule(cfg, t, 2)
            assert H.canonical([it for l in lines for it in l]) == H.canonical(R.ref_build_dump(cfg, t, 2).items)


@pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("d,k", [(96, 4), (64, 1), (130, 2)])
def test_block_diag_split_and_flops_match_reference(d, k):
    """kfac.block_diag_split_factor / inversion_flops / block_diag_inversion_flops
    vs the compiled reference (kfac.cpp:203-226), bit-exact; K must divide d."""
    import torch
    from paper_2211_14133_b200 import kfac as K
    m = R.orc_symmetric(7 + d, (d, d))
    blocks, ff, fb = R.ref_block_diag_split(m, k)
    ours = K.block_diag_split_factor(torch.from_numpy(m), k)
    assert len(ours) == k and all(np.array_equal(b, o.numpy()) for b, o in zip(blocks, ours))
    assert K.inversion_flops(d) == ff and K.block_diag_inversion_flops(d, k) == fb
    with pytest.raises(ValueError):
        K.block_diag_split_factor(torch.from_numpy(m), 7)
