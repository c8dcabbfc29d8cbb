"""Pipeline runtime (paper_2211_14133_b200/runtime.py): the per-device
programs derived from the reference assigner's FilledSchedule, checked for
conservation, communication consistency (deadlock freedom by construction)
and K-FAC dependency order; then executed for real over torch.distributed
(gloo, world size 2 and 4) with a recording test backend."""
import os
import socket
from collections import Counter

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_14133_b200 import runtime as R
from paper_2211_14133_b200 import schedule as S

CASES = [
    ("gpipe_d4n4", S.Method.GPipe, 4, 4, 1, 3),
    ("1f1b_d4n4_w2", S.Method.OneF1B, 4, 4, 2, 6),
    ("chimera_d4n4", S.Method.Chimera, 4, 4, 2, 3),
    ("chimera_d8n8", S.Method.Chimera, 8, 8, 2, 3),
    ("gpipe_d2n2_w2", S.Method.GPipe, 2, 2, 2, 1),
]
COSTS = S.CostTable(t_f=1.0, t_b=2.0, t_curv=0.05, t_inv=0.3, t_prec=0.1)


def build(method, D, N, W, L, inv_par=False, recompute=False):
    cfg = S.PipelineConfig(method=method, stages=D, micro_batches=N, micro_batch_size=32,
                           replicas=W, layers_per_stage=L, recompute=recompute)
    base = S.build_schedule(cfg, COSTS)
    filled = S.assign_works(base, cfg, COSTS, S.enumerate_kfac_works(cfg, COSTS),
                            S.AssignOptions(inversion_parallel=inv_par))
    return cfg, filled, R.device_programs(filled, cfg)  # inverse broadcast whenever W > 1


@pytest.mark.parametrize("name,method,D,N,W,L", CASES)
def test_programs_conserve_the_filled_schedule(name, method, D, N, W, L):
    cfg, filled, progs = build(method, D, N, W, L)
    assert len(progs) == cfg.effective_devices()
    for dev, (p, line) in enumerate(zip(progs, filled.schedule.timelines)):
        got = Counter(o.key() for o in p if not o.synthetic)
        want = Counter((R._KIND[w.kind], w.stage, w.micro_batch, w.layer,
                        None if w.factor is None else int(w.factor), w.step) for w in line)
        assert got == want, dev
        starts = [o.start for o in p if not o.synthetic]
        assert starts == sorted(starts)


@pytest.mark.parametrize("name,method,D,N,W,L", CASES)
def test_channels_fifo_and_collectives_ordered(name, method, D, N, W, L):
    _, _, progs = build(method, D, N, W, L)
    R.check_channel_fifo(progs)
    R.check_collective_order(progs)


@pytest.mark.parametrize("inv_par", [False, True])
def test_chimera_inversion_parallel_broadcasts_consistent(inv_par):
    _, _, progs = build(S.Method.Chimera, 4, 4, 2, 3, inv_par)
    R.check_collective_order(progs)
    n_b = sum(o.kind == "BCAST_INV" for p in progs for o in p)
    n_inv = sum(o.kind == R.INV for p in progs for o in p)
    # the reference inverts each (layer, factor) on ONE replica (the front, or
    # round-robin under inversion parallelism): every replica joins its broadcast
    assert n_b == 2 * n_inv


@pytest.mark.parametrize("name,method,D,N,W,L", CASES)
def test_kfac_dependencies_respected(name, method, D, N, W, L):
    """Curvature after its anchor F/B (gate), Sync/Inversion after the
    device's curvature of that (stage, layer, factor), Precondition after
    SyncGrad of its stage and the stage's last backward."""
    _, _, progs = build(method, D, N, W, L)
    for p in progs:
        seen_curv = Counter()
        for i, o in enumerate(p):
            if o.kind in R.KFAC_STREAM_OPS:
                assert o.gate is not None and o.gate < i and p[o.gate].kind in (R.F_, R.B_)
            if o.kind == R.CURV:
                seen_curv[(o.stage, o.layer, o.factor)] += 1
                if o.step == 0:
                    # the anchor F (A-set) / B (B-set) of this micro already ran in step 0
                    anchor = R.F_ if o.factor == 0 else R.B_
                    assert any(q.kind == anchor and q.micro == o.micro and q.stage == o.stage and q.step == 0
                               for q in p[:i])
            if o.kind in (R.SYNC_CURV, R.INV):
                later = [q for q in p[i + 1:] if q.kind == R.CURV and q.step == o.step and
                         (q.stage, q.layer, q.factor) == (o.stage, o.layer, o.factor)]
                assert not later
            if o.kind == R.PREC:
                fbs = [q for q in p[:i] if q.kind == R.B_ and q.stage == o.stage and q.step == o.step]
                assert fbs, "precondition before the stage's backward"


@pytest.mark.parametrize("method", [S.Method.GPipe, S.Method.OneF1B, S.Method.Chimera])
def test_recompute_items_run_right_before_their_backward(method):
    """With activation recomputation the reference schedule glues a Recompute
    item (duration t_f) in front of every Backward on its device
    (schedule.cpp:188-189, :215-223); the programs keep it there."""
    cfg, filled, progs = build(method, 4, 4, 2 if method == S.Method.Chimera else 1, 2, recompute=True)
    n_rec = 0
    for dev, (p, line) in enumerate(zip(progs, filled.schedule.timelines)):
        got = Counter(o.key() for o in p if not o.synthetic)
        want = Counter((R._KIND[w.kind], w.stage, w.micro_batch, w.layer,
                        None if w.factor is None else int(w.factor), w.step) for w in line)
        assert got == want, dev
        compute = [o for o in p if o.kind in R.COMPUTE_OPS]
        for i, o in enumerate(compute):
            if o.kind == R.B_:
                prev = compute[i - 1]
                assert (prev.kind, prev.stage, prev.micro, prev.step) == (R.RECOMP, o.stage, o.micro, o.step)
                assert abs(prev.start + COSTS.t_f - o.start) < 1e-9
                n_rec += 1
    assert n_rec == sum(1 for p in progs for o in p if o.kind == R.RECOMP) > 0
    R.check_channel_fifo(progs)


def test_inline_program_single_device():
    cfg = S.PipelineConfig(stages=1, micro_batches=4, layers_per_stage=24)
    prog = R.inline_program(cfg, refresh=2)
    kinds = Counter(o.kind for o in prog)
    assert kinds[R.F_] == kinds[R.B_] == 8
    assert kinds[R.CURV] == 4 * 24 * 2 and kinds[R.INV] == 24 * 2 and kinds[R.PREC] == 2
    # 1F1B on one device: F0 B0 F1 B1 ...
    fb = [(o.kind, o.micro) for o in prog if o.kind in (R.F_, R.B_) and o.step == 0]
    assert fb == [(R.F_, 0), (R.B_, 0), (R.F_, 1), (R.B_, 1), (R.F_, 2), (R.B_, 2), (R.F_, 3), (R.B_, 3)]
    # step 0: micro-batch m's curvature items right after its backward (gated on it)
    for i, o in enumerate(prog):
        if o.kind == R.CURV:
            g = prog[o.gate]
            assert (g.kind, g.micro, g.step) == (R.B_, o.micro, 0)
    inv = [i for i, o in enumerate(prog) if o.kind == R.INV]
    last_b0 = max(i for i, o in enumerate(prog) if o.kind == R.B_ and o.step == 0)
    assert min(inv) > last_b0 and all(prog[i].gate == last_b0 for i in inv)
    with pytest.raises(ValueError):
        R.inline_program(S.PipelineConfig(stages=2, micro_batches=2), 1)
    rc = R.inline_program(S.PipelineConfig(stages=1, micro_batches=3, layers_per_stage=2, recompute=True), 1)
    fb = [(o.kind, o.micro) for o in rc if o.kind in R.COMPUTE_OPS]
    assert fb == [(R.F_, 0), (R.RECOMP, 0), (R.B_, 0), (R.F_, 1), (R.RECOMP, 1), (R.B_, 1),
                  (R.F_, 2), (R.RECOMP, 2), (R.B_, 2)]


# ---------------------------------------------------------------- real execution (gloo)
class RecordingBackend:
    """Test double: F/B move tagged tensors so the receiver can verify it got
    the right micro-batch of the right stage; K-FAC ops are recorded."""

    def __init__(self, rank, topo):
        self.rank, self.topo = rank, topo
        self.recompute_on = topo.cfg.recompute
        self.log = []

    def act_shape(self, stage, micro):
        return (4,), torch.float32

    def mark_compute(self):
        return ("done", len(self.log))

    def forward(self, stage, micro, x, capture, cycle):
        if stage > 0:
            assert x.tolist() == [stage - 1, micro, 0, cycle], (stage, micro, x)
        self.log.append(("F", stage, micro))
        return torch.tensor([stage, micro, 0, cycle], dtype=torch.float32)

    def recompute(self, stage, micro):
        self.log.append(("RECOMP", stage, micro))

    def backward(self, stage, micro, gy, capture):
        if self.recompute_on:  # the micro-batch's recompute ran right before
            assert self.log[-1] == ("RECOMP", stage, micro), self.log[-3:]
        if stage < self.topo.D - 1:
            assert gy.tolist() == [stage + 1, micro, 1, 0], (stage, micro, gy)
        self.log.append(("B", stage, micro))
        return torch.tensor([stage, micro, 1, 0], dtype=torch.float32)

    def curvature(self, stage, layer, f, micro, gate):
        assert gate is not None
        self.log.append(("CURV", stage, layer, f, micro))

    def sync_curvature(self, stage, layer, f, group, gate):
        t = torch.tensor([float(self.rank)])
        dist.all_reduce(t, group=group)
        self.log.append(("SYNC_CURV", stage, layer, f, t.item()))

    def invert(self, stage, layer, f, gate):
        self.log.append(("INV", stage, layer, f))

    def broadcast_inverse(self, stage, layer, f, owner, group, gate):
        t = torch.tensor([float(self.rank)])
        dist.broadcast(t, src=owner, group=group)
        assert t.item() == owner
        self.log.append(("BCAST", stage, layer, f))

    def sync_grad(self, stage, group):
        t = torch.tensor([1.0])
        dist.all_reduce(t, group=group)
        self.log.append(("SYNC_GRAD", stage, t.item()))

    def precondition(self, stage, step):
        self.log.append(("PREC", stage, step))

    def end_cycle(self):
        pass


def _worker(rank, world, port, method, D, N, W, L, inv_par, q, recompute=False):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, filled, progs = build(method, D, N, W, L, inv_par, recompute)
        topo = R.Topology(cfg)
        comm = R.Comm(dist, rank, R.channel_plan(progs), [topo.replicas(s) for s in range(D)])
        be = RecordingBackend(rank, topo)
        ex = R.Executor(progs[rank], be, comm, rank)
        for cycle in range(2):
            ex.run_cycle(cycle)
            comm.flush()
        q.put((rank, be.log))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("method,D,N,W,L,inv_par,recompute", [
    (S.Method.GPipe, 2, 2, 1, 1, False, False),
    (S.Method.OneF1B, 2, 4, 1, 2, False, False),
    (S.Method.Chimera, 4, 4, 2, 1, False, False),   # world 4: both pipes, SyncCurvature + SyncGrad
    (S.Method.GPipe, 2, 2, 2, 1, True, False),      # world 4: data-parallel replicas, inverse broadcast
    (S.Method.OneF1B, 2, 4, 1, 2, False, True),     # activation recomputation before every backward
])
def test_gloo_execution_no_deadlock_and_data_routed(method, D, N, W, L, inv_par, recompute):
    cfg = S.PipelineConfig(method=method, stages=D, micro_batches=N, replicas=W, layers_per_stage=L,
                           recompute=recompute)
    world = cfg.effective_devices()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, method, D, N, W, L, inv_par, q, recompute))
             for r in range(world)]
    for p in procs:
        p.start()
    logs = {}
    for _ in range(world):
        r, log = q.get(timeout=120)
        logs[r] = log
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, _, progs = build(method, D, N, W, L, inv_par, recompute)
    for r in range(world):
        n_ops = sum(1 for o in progs[r])
        assert len(logs[r]) == 2 * n_ops
        syncs = [e for e in logs[r] if e[0] == "SYNC_CURV"]
        if W > 1 or method == S.Method.Chimera:
            assert syncs and all(e[-1] > 0 for e in syncs)  # every replica joined


def test_measured_costs_follow_reference_semantics():
    """engine.costs_from_times: t_curv per (layer, set, micro) item, t_inv =
    l x one set's inversion (items last t_inv / l), t_prec = per-device tail
    (spd x stage), collective volumes from the stage's bytes."""
    from paper_2211_14133_b200.engine import MeasuredTimes, costs_from_times
    t = MeasuredTimes(f=0.5, b=1.0, curv=0.1, inv=2.0, prec=0.3, layers=3, stages_per_device=2,
                      param_bytes=10 ** 8, factor_bytes=4 * 10 ** 8)
    c = costs_from_times(t)
    assert (c.t_f, c.t_b, c.t_curv, c.t_inv, c.t_prec) == (0.5, 1.0, 0.1, 6.0, 0.6)
    assert c.m_theta == 10 ** 8 and c.m_curv == 4 * 10 ** 8
    cfg = S.PipelineConfig(method=S.Method.GPipe, stages=4, micro_batches=4, replicas=1, layers_per_stage=3)
    q = S.enumerate_kfac_works(cfg, c)
    inv = [w for w in q.items if w.kind == S.WorkKind.Inversion]
    assert inv and all(abs(w.duration - c.t_inv / 3) < 1e-12 for w in inv)
    base = S.build_schedule(cfg, c)
    filled = S.assign_works(base, cfg, c, q, S.AssignOptions())
    assert filled.refresh_period >= 1


def test_pipeline_projection_from_measured_costs():
    """engine.project_pipeline: per-layer item costs -> the reference assigner
    on a D-stage config; PipeFisher period >= plain period, refresh >= 1."""
    from paper_2211_14133_b200.engine import MeasuredTimes, project_pipeline
    t = MeasuredTimes(f=12.0, b=24.0, curv=0.1, inv=1.0, prec=2.4, layers=24, stages_per_device=1,
                      param_bytes=10 ** 9, factor_bytes=10 ** 9)
    cfg = S.PipelineConfig(method=S.Method.GPipe, stages=4, micro_batches=4, micro_batch_size=32,
                           replicas=1, layers_per_stage=6, seq_len=128)
    r = project_pipeline(t, cfg)
    assert r["cost_table"]["t_f"] == 3.0 and r["cost_table"]["t_inv"] == 6.0
    assert r["pipefisher_step_ms"] >= r["plain_step_ms"] and r["refresh_period"] >= 1
    assert 0.0 < r["simulated_util"] <= 1.0


@pytest.mark.parametrize("name,method,D,N,W,L", CASES)
def test_bubble_landing_of_an_on_schedule_trace(name, method, D, N, W, L):
    """engine.bubble_landing maps each recorded K-FAC event to the bubble its
    gate names.  A trace that runs every op exactly at its schedule time (ms =
    schedule units) lands all K-FAC time inside its bubbles with no F/B
    overlap; stretching one item past the next F/B start shows up as spill."""
    from paper_2211_14133_b200.engine import bubble_landing
    _, filled, progs = build(method, D, N, W, L)
    span = filled.schedule.makespan if hasattr(filled.schedule, "makespan") else \
        max(o.start + o.duration for p in progs for o in p)
    for p in progs:
        trace = []
        for i, o in enumerate(p):
            if o.kind in (R.F_, R.B_, R.CURV, R.SYNC_CURV, R.INV):
                trace.append((o.kind, o.start, o.start + o.duration, {"op": i, "gate": o.gate}))
        rep = bubble_landing(p, trace, span)
        n_kfac = sum(o.kind in R.KFAC_STREAM_OPS for o in p)
        assert sum(b["items"] for b in rep["bubbles"]) == n_kfac
        assert rep["started_before_gate"] == 0
        if rep["kfac_ms"] > 0:
            assert rep["inside_fraction"] == pytest.approx(1.0, abs=1e-9)
            assert rep["fb_overlap_fraction"] == pytest.approx(0.0, abs=1e-9)
        for b in rep["bubbles"]:
            if b["planned"] is not None and b["next"] is not None:
                assert b["measured_ms"] == pytest.approx(b["planned"], abs=1e-9)
        # one curvature item overruns its bubble by 0.5 units
        j = next((k for k, (kind, a, b, m) in enumerate(trace)
                  if kind == R.CURV and m["gate"] is not None and
                  any(q.kind in R.COMPUTE_OPS for q in p[m["gate"] + 1:])), None)
        if j is None:
            continue
        kind, a, b, m = trace[j]
        nxt = next(i for i in range(m["gate"] + 1, len(p)) if p[i].kind in R.COMPUTE_OPS)
        trace[j] = (kind, a, p[nxt].start + 0.5, m)
        rep = bubble_landing(p, trace, span)
        spill = sum(bb["spill_ms"] for bb in rep["bubbles"])
        assert spill == pytest.approx(0.5, abs=1e-9)
        assert rep["fb_overlap_fraction"] > 0
