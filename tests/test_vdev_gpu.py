"""Multi-device PipeFisher programs executed with the PRODUCT backend
(engine.CudaBackend: BERT F/B + libpf_b200.so K-FAC kernels) on virtual
devices sharing one B200 (vdev.py: one thread and one stream set per device,
in-process P2P and collectives).  This is how the D > 1 programs of
runtime.device_programs run on the single-GPU boxes of this build.

Checks:
* GPipe D = 4 (W = 1): every rank executes its whole program; the step-0
  losses equal, bit for bit, the four stages run one after the other in one
  thread (the stage-to-stage activations arrive intact and in micro-batch
  order);
* Chimera D = 4 (its two pipes are the W = 2 replicas of every stage) with
  inversion parallelism, and 1F1B D = 2 x W = 2: every SyncCurvature
  all-reduce returns the replica average to fp32 rounding (packed lower
  triangles) and leaves the replicas bit-identical; every inverse broadcast
  delivers the owner's digit form bit for bit; SyncGrad keeps the replicas'
  weights bit-identical through the preconditioned updates.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2211_14133_b200 import schedule as S  # noqa: E402
from paper_2211_14133_b200.bert import BertConfig  # noqa: E402


def tiny(layers):
    return BertConfig(hidden=256, ffn=1024, heads=4, layers=layers, vocab=512, max_pos=128)


def run(cfg, bert, cycles=2, inversion_parallel=False, log=False, record=False):
    from paper_2211_14133_b200 import vdev
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    n = cfg.effective_devices()

    def body(rank, dist):
        with dist.init_lock:  # seeded init: one rank at a time (process-global CPU generator)
            t = PipeFisherTrainer(cfg, bert, rank=rank, world=n, kfac=True, damping=0.1, lr=1e-2, seed=3,
                                  dist=dist, inversion_parallel=inversion_parallel)
        res = []
        for _ in range(cycles):
            r = t.run_cycle(record=record)
            res.append(r)
        torch.cuda.synchronize()
        return t, res

    out, world = vdev.run_virtual(n, body, log=log)
    return out, world


def test_gpipe_d4_matches_sequential_stages():
    from paper_2211_14133_b200.bert import BertStage, synthetic_batch
    bert = tiny(8)
    cfg = S.PipelineConfig(method=S.Method.GPipe, stages=4, micro_batches=4, micro_batch_size=4, seq_len=64,
                           layers_per_stage=2)
    out, _ = run(cfg, bert, cycles=1, record=True)
    for t, res in out:  # every rank ran its program
        assert t.last_trace and res[0].cycle_ms > 0
    got = [float(x) for x in out[3][0].backend.losses[:4]]  # step 0, micro 0..3: initial weights
    # the same four stages (CudaBackend seeds stage s with seed + s) run one after
    # the other in ONE thread, the hidden state cast to bf16 between stages as the
    # pipeline sends it: the pipelined run must reproduce these losses bit for bit
    dev = torch.device("cuda")
    stages = []
    for s in range(4):
        torch.manual_seed(3 + s)
        stages.append(BertStage(bert, 2 * s, 2, s == 0, s == 3).to(dev))
    ref = []
    with torch.no_grad():
        for m in range(4):
            ids, pos, labels = synthetic_batch(bert, 4, 64, 3 + m, dev)
            x = stages[0](ids, pos, labels)
            for s in (1, 2, 3):
                x = stages[s](x.to(torch.bfloat16), pos, labels)
            ref.append(float(x))
    assert got == ref, (got, ref)


def _check_replica_collectives(world):
    n_sync = n_bcast = 0
    for c in world.collectives:
        before, after = c["before"], c["after"]
        if c["kind"] == "all_reduce" and before[0].dtype == torch.float32:
            mean = torch.stack([b.double() for b in before]).mean(0)
            for a in after:
                assert torch.equal(a, after[0])  # every replica holds the same bits
            denom = mean.abs().max().clamp_min(1e-30)
            assert float((after[0].double() - mean).abs().max() / denom) < 1e-6
            n_sync += 1
        elif c["kind"] == "broadcast":
            for a in after:
                assert torch.equal(a, after[0])
            n_bcast += 1
    return n_sync, n_bcast


def _replicas_identical(out, topo):
    for stage in range(topo.D):
        devs = topo.replicas(stage)
        ref = out[devs[0]][0].backend
        for d in devs[1:]:
            other = out[d][0].backend
            for (pa, pb) in zip(ref.stages[stage].parameters(), other.stages[stage].parameters()):
                assert torch.equal(pa, pb), f"stage {stage}: replica {d} weights differ"
            ka, kb = ref.kstate[stage], other.kstate[stage]
            for key, m in ka.factor.items():
                assert torch.equal(torch.tril(m), torch.tril(kb.factor[key])), f"factor {key} differs"
            assert ka.version == kb.version


@pytest.mark.parametrize("inversion_parallel", [False, True])
def test_chimera_d4_collectives_and_replica_consistency(inversion_parallel):
    bert = tiny(8)
    cfg = S.PipelineConfig(method=S.Method.Chimera, stages=4, micro_batches=4, micro_batch_size=4, seq_len=64,
                           layers_per_stage=2, replicas=2)
    out, world = run(cfg, bert, cycles=2, inversion_parallel=inversion_parallel, log=True)
    n_sync, n_bcast = _check_replica_collectives(world)
    assert n_sync > 0
    assert n_bcast > 0  # each inverse goes from its one inverting replica to the other
    topo = out[0][0].topo
    _replicas_identical(out, topo)
    for stage in range(topo.D):  # the digit-form inverses the preconditioner reads agree too
        devs = topo.replicas(stage)
        ka = out[devs[0]][0].backend.kstate[stage]
        for d in devs[1:]:
            kb = out[d][0].backend.kstate[stage]
            for key, m in ka.inv.items():
                assert torch.equal(m.digits, kb.inv[key].digits), f"inverse digits {key} differ on {d}"
    for t, res in out:
        assert all(r.loss is None or torch.isfinite(torch.tensor(r.loss)) for r in res)


def test_1f1b_d2_w2_data_parallel():
    bert = tiny(4)
    cfg = S.PipelineConfig(method=S.Method.OneF1B, stages=2, micro_batches=4, micro_batch_size=4, seq_len=64,
                           layers_per_stage=2, replicas=2)
    out, world = run(cfg, bert, cycles=2, log=True)
    n_sync, _ = _check_replica_collectives(world)
    assert n_sync > 0
    # W = 2 data-parallel groups see DIFFERENT data, yet SyncCurvature and
    # SyncGrad make every stage's replicas identical after each cycle
    _replicas_identical(out, out[0][0].topo)


def test_chimera_d4_kfac_landing_recorded():
    """Where the K-FAC items land against their assigned bubbles (measured CUDA
    events of a recorded cycle, engine.bubble_landing): every item accounted
    for, none starts before the F/B op it is gated on.  The virtual devices
    share one GPU's SMs, so the lengths are not a multi-GPU measurement; with
    PF_LANDING_OUT set the per-rank reports are written there as JSON."""
    import json
    import os
    from paper_2211_14133_b200 import runtime as R
    from paper_2211_14133_b200.engine import trainer_bubble_landing
    bert = tiny(8)
    cfg = S.PipelineConfig(method=S.Method.Chimera, stages=4, micro_batches=4, micro_batch_size=4, seq_len=64,
                           layers_per_stage=2, replicas=2)
    out, _ = run(cfg, bert, cycles=2, record=True)
    reports = []
    for t, res in out:
        rep = trainer_bubble_landing(t)
        n_kfac = sum(o.kind in R.KFAC_STREAM_OPS for o in t.program)
        assert sum(b["items"] for b in rep["bubbles"]) == n_kfac
        assert rep["started_before_gate"] == 0
        assert 0.0 <= rep["inside_fraction"] <= 1.0
        reports.append({"rank": t.rank, "cycle_ms": t.last_cycle_ms, **rep})
    path = os.environ.get("PF_LANDING_OUT")
    if path:
        with open(path, "w") as f:
            json.dump({"config": "Chimera D=4 W=2 (virtual devices on one B200), tiny BERT", "ranks": reports},
                      f, indent=1)
