"""GPU parity of the K-FAC kernels (through the C-ABI) with the oracle.

Tolerances (BASELINE.json north_star):
  factors              relative Frobenius <= 1e-3 vs the FP64 oracle on the SAME
                       bf16-rounded inputs (measured ~1e-6: fp32 accumulation only)
  damped inverse       max |(M + lambda I) X - I| <= 1e-5   (reference norm,
                       proj/tests/test_kfac.cpp:155), plus rel. Frobenius vs oracle
  precondition/update  relative Frobenius <= 1e-3 vs oracle (3xTF32 gives ~1e-6)
Oracle = oracle/kfac_oracle.c (bit-identical to the compiled reference, see
tests/test_oracle.py) for sizes it finishes in seconds; at BASELINE sizes
(d = 3072/4096) size-independent properties are checked instead
(residual of the inverse, symmetry, agreement with an fp64 torch product).
"""
import numpy as np
import pytest
import torch

from oracle import ref as R

pytestmark = pytest.mark.gpu

FACTOR_TOL = 1e-3
INV_RESIDUAL_TOL = 1e-5
PREC_TOL = 1e-3


@pytest.fixture(scope="module")
def K():
    assert torch.cuda.is_available(), "gpu tests need a CUDA device"
    from paper_2211_14133_b200 import kfac
    assert kfac.device_ok(), "libpf_b200.so needs an sm_100 device"
    return kfac


def rel_fro(got, want):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))


def bf16_tape(seed, d, n):
    """SplitMix64 unit-variance inputs, rounded to bf16; returns
    (device bf16 tensor, the same values as fp64 numpy for the oracle)."""
    x = R.orc_symmetric(seed, (d, n), 3 ** 0.5)
    t = torch.from_numpy(x).to(torch.bfloat16)
    return t.cuda(), t.to(torch.float64).numpy()


def spd(seed, d, n=None):
    n = n or max(2 * d, 64)
    _, x = bf16_tape(seed, d, n)
    return (x @ x.T) / n


# ------------------------------------------------------------------ curvature
@pytest.mark.parametrize("d,n", [(64, 96), (128, 128), (200, 72), (256, 512), (384, 4096),
                                 (768, 1024), (1000, 328)])
def test_syrk_matches_oracle(K, d, n):
    x, x64 = bf16_tape(100 + d, d, n)
    f = torch.empty((d, d), dtype=torch.float32, device="cuda")
    K.syrk([(x, f, 1.0 / n, False)])
    got = f.cpu().numpy()
    want = R.orc_curvature_factor(x64)
    assert rel_fro(got, want) <= FACTOR_TOL
    assert rel_fro(got, want) <= 1e-5  # fp32 accumulation only
    assert np.array_equal(got, got.T)


def test_curvature_factors_api_matches_reference_call(K):
    """kfac::curvature_factors on a one-layer tape, A and B in one launch."""
    a, a64 = bf16_tape(7, 96, 160)
    e, e64 = bf16_tape(8, 40, 160)
    tape = K.BatchTape([a], [e], 160)
    A, B = K.curvature_factors(tape, 0)
    RA, RB = R.ref_curvature_factors(a64, e64)
    assert rel_fro(A.cpu().numpy(), RA) <= 1e-5
    assert rel_fro(B.cpu().numpy(), RB) <= 1e-5


def test_syrk_accumulate_lower_only_and_grouped(K):
    x1, x1_64 = bf16_tape(1, 256, 256)
    x2, x2_64 = bf16_tape(2, 256, 256)
    f = torch.full((256, 256), 7.0, device="cuda")
    K.syrk([(x1, f, 0.5, False)], fill_upper=False)
    K.syrk([(x2, f, 0.25, True)], fill_upper=False)
    want = 0.5 * (x1_64 @ x1_64.T) + 0.25 * (x2_64 @ x2_64.T)
    got = f.cpu().numpy()
    il = np.tril_indices(256)
    assert rel_fro(got[il], want[il]) <= 1e-5
    # grouped: three different sizes in one launch
    xs = [bf16_tape(10 + i, d, 512) for i, d in enumerate((128, 768, 3072))]
    fs = [torch.empty((d, d), device="cuda") for d in (128, 768, 3072)]
    K.syrk([(x, f, 1 / 512, False) for (x, _), f in zip(xs, fs)])
    for (x, x64), f in zip(xs, fs):
        ref = torch.from_numpy(x64).cuda()
        want = (ref @ ref.T) / 512
        assert rel_fro(f.double().cpu().numpy(), want.cpu().numpy()) <= 1e-5


@pytest.mark.parametrize("d", [1024, 4096])
def test_syrk_baseline_sizes(K, d):
    """n = 32 x 128 = 4096 tokens; checked against an fp64 product (same bf16 inputs)."""
    x, _ = bf16_tape(77 + d, d, 4096)
    f = torch.empty((d, d), device="cuda")
    K.syrk([(x, f, 1 / 4096, False)])
    xd = x.double()
    want = (xd @ xd.T) / 4096
    assert torch.linalg.norm(f.double() - want) / torch.linalg.norm(want) <= 1e-5
    assert torch.equal(f, f.T)


# ------------------------------------------------------------------ inverse
def residual(m64, inv64, lam):
    a = torch.from_numpy(m64).cuda() + lam * torch.eye(m64.shape[0], dtype=torch.float64, device="cuda")
    x = torch.from_numpy(inv64).cuda()
    return float((a @ x - torch.eye(m64.shape[0], dtype=torch.float64, device="cuda")).abs().max())


@pytest.mark.parametrize("d", [1, 32, 100, 128, 129, 256, 300, 512, 768, 1024])
def test_damped_inverse_matches_oracle(K, d):
    m = spd(300 + d, d)
    lam = 0.1
    got = K.cholesky_spd_inverse(torch.from_numpy(m).float().cuda(), lam).double().cpu().numpy()
    m32 = m.astype(np.float32).astype(np.float64)  # the kernel's input
    want = R.orc_cholesky_spd_inverse(m32, lam)
    assert rel_fro(got, want) <= 1e-4
    assert residual(m32, got, lam) <= INV_RESIDUAL_TOL
    assert np.abs(got - got.T).max() == 0.0


@pytest.mark.parametrize("d", [2048, 3072, 4096])
def test_damped_inverse_residual_baseline_sizes(K, d):
    x, _ = bf16_tape(900 + d, d, 4096)
    f = torch.empty((d, d), device="cuda")
    K.syrk([(x, f, 1 / 4096, False)])
    inv = K.cholesky_spd_inverse(f, 0.1)
    a = f.double() + 0.1 * torch.eye(d, dtype=torch.float64, device="cuda")
    r = float((a @ inv.double() - torch.eye(d, dtype=torch.float64, device="cuda")).abs().max())
    assert r <= INV_RESIDUAL_TOL


def test_damped_inverse_batched_mixed_sizes_and_digits(K):
    ms = [spd(40 + i, d) for i, d in enumerate((64, 768, 768, 1024))]
    ts = [torch.from_numpy(m).float().cuda() for m in ms]
    outs = [torch.empty_like(t) for t in ts]
    digits = [torch.empty(K.slice_bytes(t.shape[0], t.shape[0]), dtype=torch.uint8, device="cuda")
              for t in ts]
    K.damped_inverse_batched(ts, 0.1, outs, digits)
    single = [K.cholesky_spd_inverse(t, 0.1) for t in ts]
    for m, o, s1 in zip(ms, outs, single):
        assert torch.equal(o, s1)  # batching does not change the arithmetic
        m32 = m.astype(np.float32).astype(np.float64)
        assert residual(m32, o.double().cpu().numpy(), 0.1) <= INV_RESIDUAL_TOL
    # digit form reproduces the fp32 inverse to 2^-27 of each row's scale
    sl = K.slice_matrix(outs[1])
    assert torch.equal(sl.digits, digits[1])


def test_not_positive_definite_raises_with_column(K):
    """proj/tests/test_kfac.cpp:158-160: [[1,2],[2,1]] is indefinite."""
    with pytest.raises(K.NotPositiveDefinite) as e:
        K.cholesky_spd_inverse(torch.tensor([[1.0, 2.0], [2.0, 1.0]], device="cuda"), 0.0)
    assert e.value.column == 2
    with pytest.raises(R.DomainError):
        R.orc_cholesky_spd_inverse(np.array([[1.0, 2.0], [2.0, 1.0]]), 0.0)
    m = np.eye(300)
    m[170, 170] = -1.0
    with pytest.raises(K.NotPositiveDefinite) as e:
        K.cholesky_spd_inverse(torch.from_numpy(m).float().cuda(), 0.5)
    assert e.value.column == 171


def test_inverse_hand_cases(K):
    got = K.cholesky_spd_inverse(torch.tensor([[4.0, 0.0], [0.0, 9.0]], device="cuda"), 0.0)
    assert torch.allclose(got, torch.tensor([[0.25, 0.0], [0.0, 1 / 9]], device="cuda"), atol=1e-7)
    assert torch.equal(K.cholesky_spd_inverse(torch.eye(3, device="cuda"), 0.0),
                       torch.eye(3, device="cuda"))


# ------------------------------------------------------------------ precondition
@pytest.mark.parametrize("d_out,d_in", [(1, 2), (40, 96), (128, 128), (256, 768), (768, 256),
                                        (768, 768), (300, 200)])
def test_precondition_matches_oracle(K, d_out, d_in):
    ai = np.linalg.inv(spd(1, d_in) + 0.1 * np.eye(d_in))
    bi = np.linalg.inv(spd(2, d_out) + 0.1 * np.eye(d_out))
    g = R.orc_symmetric(3, (d_out, d_in))
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).float().cuda()
    got = K.precondition(t(g), t(ai), t(bi)).double().cpu().numpy()
    want = R.orc_precondition(g.astype(np.float32).astype(np.float64),
                              ai.astype(np.float32).astype(np.float64),
                              bi.astype(np.float32).astype(np.float64))
    assert rel_fro(got, want) <= PREC_TOL
    assert rel_fro(got, want) <= 1e-6  # digit-form GEMMs: ~fp32 rounding only


def test_precondition_hand_case(K):
    """proj/tests/test_kfac.cpp:162-169."""
    g = torch.tensor([[6.0, 6.0]], device="cuda")
    got = K.precondition(g, 0.5 * torch.eye(2, device="cuda"), torch.tensor([[1 / 3]], device="cuda"))
    assert torch.allclose(got, torch.tensor([[1.0, 1.0]], device="cuda"), atol=1e-6)
    with pytest.raises(ValueError):
        K.precondition(g, torch.eye(3, device="cuda"), torch.tensor([[1 / 3]], device="cuda"))


@pytest.mark.parametrize("d_out,d_in", [(4096, 1024), (1024, 4096), (1000, 2504), (2300, 700)])
def test_precondition_update_baseline_sizes(K, d_out, d_in):
    """Fused W -= eta B^-1 G A^-1 at BERT-Large FFN shapes vs an fp64 torch product."""
    torch.manual_seed(0)
    ai = torch.randn(d_in, d_in, device="cuda", dtype=torch.float64) / d_in ** 0.5
    ai = (ai @ ai.T + 0.1 * torch.eye(d_in, device="cuda", dtype=torch.float64)).float()
    bi = torch.randn(d_out, d_out, device="cuda", dtype=torch.float64) / d_out ** 0.5
    bi = (bi @ bi.T + 0.1 * torch.eye(d_out, device="cuda", dtype=torch.float64)).float()
    g = torch.randn(d_out, d_in, device="cuda")
    w = 0.02 * torch.randn(d_out, d_in, device="cuda")
    want = w.double() - 1e-3 * (bi.double() @ g.double() @ ai.double())
    w2 = w.clone()
    K.precondition_update(w2, g, ai, bi, 1e-3)
    delta_got = (w2.double() - w.double())
    delta_want = want - w.double()
    assert float(torch.linalg.norm(delta_got - delta_want) / torch.linalg.norm(delta_want)) <= 1e-5


def test_precondition_batched_mixed_long_k(K):
    """One batched call mixing K = 1024 and K = 4096 products (the BERT-Large
    layer mix, run by the persistent long-K GEMM with its tile queue) equals
    the per-problem calls bit for bit and an fp64 product to 1e-5."""
    torch.manual_seed(1)
    shapes = [(1024, 1024), (1024, 1024), (4096, 1024), (1024, 4096)]
    items, singles, wants = [], [], []
    for d_out, d_in in shapes:
        ai = torch.randn(d_in, d_in, device="cuda", dtype=torch.float64) / d_in ** 0.5
        ai = (ai @ ai.T + 0.1 * torch.eye(d_in, device="cuda", dtype=torch.float64)).float()
        bi = torch.randn(d_out, d_out, device="cuda", dtype=torch.float64) / d_out ** 0.5
        bi = (bi @ bi.T + 0.1 * torch.eye(d_out, device="cuda", dtype=torch.float64)).float()
        g = torch.randn(d_out, d_in, device="cuda")
        w = 0.02 * torch.randn(d_out, d_in, device="cuda")
        wants.append(-1e-3 * (bi.double() @ g.double() @ ai.double()))
        a_s, b_s = K.slice_matrix(ai), K.slice_matrix(bi)
        w1 = w.clone()
        K.precondition_update_sliced([(w1, g, a_s, b_s, 1e-3)])
        singles.append((w, w1))
        items.append((w.clone(), g, a_s, b_s, 1e-3))
    K.precondition_update_sliced(items)
    for (w, w1), (w2, *_), want in zip(singles, items, wants):
        assert torch.equal(w2, w1)
        d = w2.double() - w.double()
        assert float(torch.linalg.norm(d - want) / torch.linalg.norm(want)) <= 1e-5


def test_ngd_step_matches_reference(K):
    """kfac::ngd_step: first step plain gradient (+flag), then preconditioned."""
    d_in, d_out, n = 96, 64, 256
    a, a64 = bf16_tape(21, d_in, n)
    e, e64 = bf16_tape(22, d_out, n)
    g64 = R.orc_symmetric(23, (d_out, d_in))
    w64 = R.orc_symmetric(24, (d_out, d_in), 0.02)
    st = K.KfacState(1, damping=0.1, learning_rate=1e-2)
    w = torch.from_numpy(w64).float().cuda()
    g = torch.from_numpy(g64).float().cuda()
    r = K.ngd_step([w], st, [g])
    assert r.used_plain_gradient and st.staleness == [1]
    w_ref, plain = R.ref_ngd_step(w64.astype(np.float32).astype(np.float64),
                                  g64.astype(np.float32).astype(np.float64), None, None, 1e-2)
    assert plain and rel_fro(w.double().cpu().numpy(), w_ref) <= 1e-6
    st.update_factors(K.BatchTape([a], [e], n))
    st.refresh_inverses()
    w_before = w.double().cpu().numpy()
    r = K.ngd_step([w], st, [g])
    assert not r.used_plain_gradient and st.staleness == [1]
    A, B = R.ref_curvature_factors(a64, e64)
    Ai = R.ref_cholesky_spd_inverse(A, 0.1)
    Bi = R.ref_cholesky_spd_inverse(B, 0.1)
    w_ref, _ = R.ref_ngd_step(w_before, g64.astype(np.float32).astype(np.float64), Ai, Bi, 1e-2)
    delta = w.double().cpu().numpy() - w_before
    assert rel_fro(delta, w_ref - w_before) <= 1e-4
    K.ngd_step([w], st, [g])
    assert st.staleness == [2]


def _mixed_batch(K, sizes, seed0):
    ms = [spd(seed0 + i, d) for i, d in enumerate(sizes)]
    ts = [torch.from_numpy(m).float().cuda() for m in ms]
    outs = [torch.empty_like(t) for t in ts]
    digits = [torch.empty(K.slice_bytes(t.shape[0], t.shape[0]), dtype=torch.uint8, device="cuda") for t in ts]
    return ms, ts, outs, digits


@pytest.mark.parametrize("sizes", [(1,), (100,), (128, 129), (256, 300, 300), (64, 768, 768, 1024), (2048, 512)])
def test_inverse_repeatable_bit_identical(K, sizes):
    """Two calls on the same inputs give bit-identical inverses and digit
    forms (fixed launch order, exact integer digit products, no atomics in
    the arithmetic), and every inverse meets the residual bound."""
    ms, ts, outs, digits = _mixed_batch(K, sizes, 70)
    K.damped_inverse_batched(ts, 0.1, outs, digits)
    ref = [(o.clone(), dg.clone()) for o, dg in zip(outs, digits)]
    for o in outs:
        o.fill_(float("nan"))
    K.damped_inverse_batched(ts, 0.1, outs, digits)
    for (o_ref, d_ref), o, dg, m in zip(ref, outs, digits, ms):
        assert torch.equal(o, o_ref)
        assert torch.equal(dg, d_ref)
        m32 = m.astype(np.float32).astype(np.float64)
        assert residual(m32, o.double().cpu().numpy(), 0.1) <= INV_RESIDUAL_TOL


def test_inverse_not_pd_columns(K):
    m = torch.tensor([[1.0, 2.0], [2.0, 1.0]], device="cuda")
    with pytest.raises(K.NotPositiveDefinite) as e:
        K.cholesky_spd_inverse(m, 0.0)
    assert e.value.column == 2
    m = np.eye(300)
    m[170, 170] = -1.0
    with pytest.raises(K.NotPositiveDefinite) as e:
        K.cholesky_spd_inverse(torch.from_numpy(m).float().cuda(), 0.5)
    assert e.value.column == 171


def test_inverse_in_cuda_graph(K):
    _, ts, outs, digits = _mixed_batch(K, (512, 256), 90)
    K.damped_inverse_batched(ts, 0.1, outs, digits, check=False)
    torch.cuda.synchronize()
    want = [o.clone() for o in outs]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            K.damped_inverse_batched(ts, 0.1, outs, digits, check=False)
    for o in outs:
        o.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert torch.equal(o, w)


@pytest.mark.parametrize("d,k", [(1024, 4), (512, 2), (384, 3)])
def test_block_diag_inverse_matches_reference_blocks(K, d, k):
    """Block-diagonal damped inverse (kfac.cpp:203-226): every diagonal block
    equals the reference cholesky_spd_inverse of the reference's
    block_diag_split_factor block; the off-diagonal blocks are exactly zero;
    the digit form reproduces the assembled inverse."""
    m = spd(500 + d, d)
    lam = 0.1
    t = torch.from_numpy(m).float().cuda()
    dg = torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda")
    (got,) = K.damped_inverse_block_diag([t], lam, k, digits=[dg])
    got = got.double().cpu().numpy()
    m32 = m.astype(np.float32).astype(np.float64)
    blocks, _, _ = R.ref_block_diag_split(m32, k)
    b = d // k
    for i, blk in enumerate(blocks):
        want = R.ref_cholesky_spd_inverse(blk, lam)
        assert rel_fro(got[i * b:(i + 1) * b, i * b:(i + 1) * b], want) <= 1e-4
        for j in range(k):
            if j != i:
                assert np.all(got[i * b:(i + 1) * b, j * b:(j + 1) * b] == 0.0)
    assert torch.equal(K.slice_matrix(torch.from_numpy(got).float().cuda()).digits, dg)


def test_kfac_state_block_diag_refresh(K):
    st = K.KfacState(1, damping=0.1, learning_rate=1e-3, block_diag_k=2)
    st.factor_a[0] = torch.from_numpy(spd(3, 256)).float().cuda()
    st.factor_b[0] = torch.from_numpy(spd(4, 100)).float().cuda()  # 2 does divide: block-diag too
    st.refresh_inverses()
    a = st.inv_a[0].fp32
    assert torch.all(a[:128, 128:] == 0) and torch.all(a[128:, :128] == 0)
    assert st.has_inverses(0) and st.staleness[0] == 0


def test_large_batch_uses_recursive_schedule_and_matches_oracle(K):
    """>= 24 factors per call switch to the throughput schedule (recursive
    blocked Cholesky); every inverse still matches the FP64 oracle."""
    sizes = [300, 256, 129] * 8  # 24 problems
    ms = [spd(1200 + i, d) for i, d in enumerate(sizes)]
    ts = [torch.from_numpy(m).float().cuda() for m in ms]
    outs = K.damped_inverse_batched(ts, 0.1)
    for m, o in zip(ms, outs):
        m32 = m.astype(np.float32).astype(np.float64)
        got = o.double().cpu().numpy()
        assert rel_fro(got, R.orc_cholesky_spd_inverse(m32, 0.1)) <= 1e-4
        assert residual(m32, got, 0.1) <= INV_RESIDUAL_TOL


@pytest.mark.parametrize("d,n", [(64, 96), (128, 128), (200, 72), (256, 512), (1024, 4096), (4096, 512)])
def test_syrk_token_major_matches_feature_major(K, d, n):
    """Token-major tapes ([n x d], a layer's activations as produced) are read
    in place as MN-major tensor-core operands: the factor is bit-identical to
    the feature-major call on the transposed copy (same bf16 products, same
    fp32 accumulation order per tile), and matches the oracle."""
    g = torch.Generator(device="cuda").manual_seed(d * 7 + n)
    xt = torch.randn((n, (d + 7) // 8 * 8), generator=g, device="cuda").to(torch.bfloat16)[:, :d]
    x = xt.t().contiguous()
    if n % 8:
        x = K.to_tape_layout(x)
    f_km = torch.empty((d, d), device="cuda")
    f_mn = torch.empty((d, d), device="cuda")
    K.syrk([(x, f_km, 1.0 / n, False)], fill_upper=True)
    K.syrk([(xt, f_mn, 1.0 / n, False, True)], fill_upper=True)
    torch.cuda.synchronize()
    assert torch.equal(f_km, f_mn)
    if d <= 256:
        want = R.orc_curvature_factor(x.double().cpu().numpy()[:, :n])
        got = f_mn.double().cpu().numpy()
        assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-3


def test_syrk_token_major_grouped_accumulate_with_padded_rows(K):
    """Grouped token-major problems with a row pitch wider than d (a view of a
    wider activation buffer) and accumulate=True."""
    g = torch.Generator(device="cuda").manual_seed(5)
    buf = torch.randn((512, 1040), generator=g, device="cuda").to(torch.bfloat16)
    a, b = buf[:, :1024], buf[:, 8:8 + 384]
    fa = torch.zeros((1024, 1024), device="cuda")
    fb = torch.full((384, 384), 0.5, device="cuda")
    K.syrk([(a, fa, 1.0, False, True), (b, fb, 2.0, True, True)], fill_upper=True)
    torch.cuda.synchronize()
    wa = a.float().t() @ a.float()
    wb = 0.5 + 2.0 * (b.float().t() @ b.float())
    assert ((fa - wa).norm() / wa.norm()).item() < 1e-5
    assert ((fb - wb).norm() / wb.norm()).item() < 1e-5


def test_graphs_captured_after_eager_calls_survive_workspace_growth(K):
    """A batched inversion run eagerly and then captured as a CUDA graph on the
    same stream, followed by a bigger batch that grows the workspace arena:
    replaying the first graph must still find its workspace (the arena keeps
    replaced buffers alive) and reproduce the eager result bit for bit."""
    s = torch.cuda.Stream()

    def mk(n, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        mats = []
        for d in [256] * n + [512]:
            x = torch.randn((d, 1024), generator=g, device="cuda").to(torch.bfloat16).float()
            mats.append(x @ x.T / 1024)
        outs = [torch.empty_like(m) for m in mats]
        digs = [torch.empty(K.slice_bytes(m.shape[0], m.shape[0]), dtype=torch.uint8, device="cuda") for m in mats]
        return mats, outs, digs

    sets = [mk(2, 1), mk(5, 2)]
    graphs, eager = [], []
    for mats, outs, digs in sets:
        with torch.cuda.stream(s):
            K.damped_inverse_batched(mats, 0.1, outs, digs, check=False)
        torch.cuda.synchronize()
        eager.append([o.clone() for o in outs])
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            K.damped_inverse_batched(mats, 0.1, outs, digs, check=False)
        graphs.append(g)
    for (mats, outs, digs), g, want in zip(sets, graphs, eager):
        for o in outs:
            o.zero_()
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        for o, w in zip(outs, want):
            assert torch.equal(o, w)
