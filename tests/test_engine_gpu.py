"""PipeFisher trainer on the B200 (engine.py + runtime.py): a small BERT run
through the single-device inline K-FAC program, with the K-FAC state checked
against an FP64 torch restatement of the reference formulas on the same
bf16 tapes (kfac.cpp:125-137, :186-201)."""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2211_14133_b200 import schedule as S  # noqa: E402
from paper_2211_14133_b200.bert import BertConfig  # noqa: E402


def small():
    return BertConfig(hidden=256, ffn=1024, heads=4, layers=2, vocab=512, max_pos=128)


def trainer(kfac=True, refresh=2, micro=2):
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    cfg = S.PipelineConfig(stages=1, micro_batches=micro, micro_batch_size=4, seq_len=64, layers_per_stage=2)
    return PipeFisherTrainer(cfg, small(), kfac=kfac, refresh=refresh, damping=0.1, lr=1e-2, seed=3)


def rel(a, b):
    return float((a.double() - b.double()).norm() / b.double().norm())


def test_inline_kfac_cycles_run_and_refresh_inverses():
    t = trainer()
    ks = t.backend.kstate[0]
    r0 = t.run_cycle(record=True)
    assert r0.loss is not None and torch.isfinite(torch.tensor(r0.loss))
    assert all(v == 0 for v in ks.version.values())  # one refresh per cycle
    assert 0.0 < r0.util <= 1.0
    for _ in range(2):
        r = t.run_cycle()
    assert all(v == 2 for v in ks.version.values())
    assert torch.isfinite(torch.tensor(r.loss))


def test_curvature_accumulates_micro_batches_like_the_reference():
    t = trainer(micro=2)
    b = t.backend
    for m in range(2):  # step-0 F/B of both micro-batches, tapes captured
        b.forward(0, m, None, True, 0)
        b.backward(0, m, None, True)
    store = b.stages[0].store
    tapes = {k: v.clone() for k, v in store.tapes.items()}
    b.curvature_many([(0, l, f, m) for m in range(2) for l in range(2) for f in (0, 1)], None)
    torch.cuda.synchronize()
    n = b.tokens * 2
    ks = b.kstate[0]
    for l in range(2):
        for key in ("a_qkv", "a_ffn2", "e_q", "e_ffn1"):
            # tapes are token-major [n x d] (read in place by the SYRK)
            want = sum(tapes[(l, key, m)].double().T @ tapes[(l, key, m)].double() for m in range(2)) / n
            got = torch.tril(ks.factor[(l, key)].double())
            assert rel(got, torch.tril(want)) < 1e-3, (l, key)


def test_inversion_and_fused_update_match_fp64():
    t = trainer(micro=2)
    b = t.backend
    t.run_cycle()  # factors + inverses of cycle 0, weights updated
    ks = b.kstate[0]
    lam = 0.1
    for l, key in ((0, "a_qkv"), (1, "e_ffn1")):
        A = torch.tril(ks.factor[(l, key)].double())
        A = A + torch.tril(A, -1).T + lam * torch.eye(A.shape[0], dtype=torch.float64, device=A.device)
        X = ks.inv[(l, key, 0)].fp32.double()
        res = (A @ X - torch.eye(A.shape[0], dtype=torch.float64, device=A.device)).abs().max().item()
        assert res < 1e-5, (l, key, res)
    # one more step's update through the engine vs FP64 on the same inverses
    layer = b.stages[0].layers[0]
    w0 = layer.w["ffn1"].detach().clone()
    b.forward(0, 0, None, False, 1)
    b.backward(0, 0, None, False)
    g = layer.w["ffn1"].grad.detach().clone()
    ai, bi = ks.inv[(0, "a_ffn1", 0)].fp32.double(), ks.inv[(0, "e_ffn1", 0)].fp32.double()
    b.precondition(0, 1)
    torch.cuda.synchronize()
    want = w0.double() - b.lr * (bi @ g.double() @ ai)
    got = layer.w["ffn1"].detach().double()
    assert rel(got - w0.double(), want - w0.double()) < 1e-3


def test_plain_pipeline_baseline_has_no_kfac_ops():
    t = trainer(kfac=False)
    assert {o.kind for o in t.program} <= {"F", "B", "SYNC_GRAD", "PREC"}
    r = t.run_cycle(record=True)
    assert torch.isfinite(torch.tensor(r.loss))


def test_measured_cost_table_closed_loop():
    """costs='measured': the work items are timed on this GPU and the cost
    table the assigner sees is built from them."""
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    cfg = S.PipelineConfig(stages=1, micro_batches=2, micro_batch_size=4, seq_len=64, layers_per_stage=2)
    t = PipeFisherTrainer(cfg, small(), kfac=True, refresh=2, costs="measured", damping=0.1, lr=1e-2, seed=3)
    m = t.measured
    assert m is not None and min(m.f, m.b, m.curv, m.inv, m.prec) > 0.0
    assert t.costs.t_inv == pytest.approx(2 * m.inv) and t.costs.t_curv == m.curv
    r = t.run_cycle(record=True)
    assert torch.isfinite(torch.tensor(r.loss))


def test_recompute_gives_the_same_training_step():
    """Activation recomputation (reference WorkKind::Recompute, schedule.cpp:
    188-189, :215-223): F keeps only the stage input, the Recompute op rebuilds
    the graph right before B.  Same losses, tapes, factors and updated weights
    as the run that keeps its activations (the recomputed forward is the same
    arithmetic), and the program carries one Recompute per backward."""
    from paper_2211_14133_b200 import runtime as R
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    runs = []
    for rc in (False, True):
        cfg = S.PipelineConfig(stages=1, micro_batches=2, micro_batch_size=4, seq_len=64, layers_per_stage=2,
                               recompute=rc)
        t = PipeFisherTrainer(cfg, small(), kfac=True, refresh=2, damping=0.1, lr=1e-2, seed=3)
        n_rec = sum(1 for o in t.program if o.kind == R.RECOMP)
        assert n_rec == (2 * 2 if rc else 0)  # refresh 2 steps x 2 micro-batches
        losses = [t.run_cycle().loss for _ in range(2)]
        torch.cuda.synchronize()
        ks = t.backend.kstate[0]
        runs.append((losses, {k: v.clone() for k, v in ks.factor.items()},
                     [p.detach().clone() for p in t.backend.stages[0].parameters()]))
    (l0, f0, w0), (l1, f1, w1) = runs
    assert l0 == l1
    for k in f0:
        assert torch.equal(f0[k], f1[k]), k
    for a, b in zip(w0, w1):
        assert torch.allclose(a, b, rtol=0, atol=1e-6)


def test_graphed_fb_gives_the_same_training_step():
    """F/B of every (stage, micro-batch, tape capture) as CUDA graphs
    (CudaBackend(graph_fb=True)): the same kernels replayed, so the same
    losses, factors and updated weights as the eager run, bit for bit."""
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    runs = []
    for gfb in (False, True):
        cfg = S.PipelineConfig(stages=1, micro_batches=2, micro_batch_size=4, seq_len=64, layers_per_stage=2)
        t = PipeFisherTrainer(cfg, small(), kfac=True, refresh=2, damping=0.1, lr=1e-2, seed=3, graph_fb=gfb)
        losses = [t.run_cycle().loss for _ in range(3)]
        torch.cuda.synchronize()
        ks = t.backend.kstate[0]
        runs.append((losses, {k: v.clone() for k, v in ks.factor.items()},
                     [p.detach().clone() for p in t.backend.stages[0].parameters()]))
        if gfb:
            assert len(t.backend.graphed) == 4  # 2 micro-batches x (tape capture on / off)
    (l0, f0, w0), (l1, f1, w1) = runs
    assert l0 == l1
    for k in f0:
        assert torch.equal(f0[k], f1[k]), k
    for a, b in zip(w0, w1):
        assert torch.equal(a, b)
