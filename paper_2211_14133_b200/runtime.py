"""PipeFisher pipeline runtime: executes a FilledSchedule (the reference
assigner's output, bit-exact — paper_2211_14133_b200/schedule.py) on real
devices.  The reference only simulates this; the design
follows SURVEY Appendix D.4.

One process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU
tests).  Per device:

* ``compute`` stream: Forward / Backward of the stages it hosts, stage-to-
  stage activations and errors over P2P, SyncGrad and Precondition (the tail);
* ``kfac`` stream (low priority): Curvature, SyncCurvature, Inversion.  Each
  K-FAC item waits on the event of the F/B op that precedes it in the
  device's timeline, so it runs in the bubble after that op and an overrun
  never delays F/B (nothing on the compute stream waits for curvature).

Correct-by-construction communication:

* P2P channels are keyed (src, dst, pipe, act|grad); on a channel both sides
  issue their ops in micro-batch order (F and B of one pipe run in micro
  order on every stage), so the FIFO pairing always matches.  Each channel
  is its own 2-rank group (its own NCCL communicator and stream): no
  cross-channel head-of-line blocking.
* Collectives of a replica group (SyncCurvature, SyncGrad, inverse
  broadcast) are issued by every member in one canonical order (the front
  device's schedule order).  The reference models SyncCurvature on the front
  replica only; the other replicas join right after their own
  last curvature item of that (layer, factor).
* Sends are asynchronous and every rank walks its program in schedule-time
  order, so a recv never waits on something its peer can only do later.

K-FAC state: curvature items of a cycle accumulate into the factors from the
step-0 tapes; inversions write a double-buffered inverse (fp32 +
digit form); a Precondition uses the newest inverse whose Inversion precedes
it in the device's program — the deterministic rule of D.4 that reproduces
``staleness_report`` — or the plain gradient before the first inverse exists
(A.13).

Single device (D = 1) has no bubbles (reference test_schedule.cpp:69-75);
``inline_program`` builds the "K-FAC + skip" step instead: F/B, then every R
steps curvature + inversion, every step precondition.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import schedule as S
from .schedule import Factor, Method, WorkKind

# ---------------------------------------------------------------------- programs
F_, B_, CURV, SYNC_CURV, INV, SYNC_GRAD, PREC = "F", "B", "CURV", "SYNC_CURV", "INV", "SYNC_GRAD", "PREC"
RECOMP = "RECOMP"
COMPUTE_OPS = (F_, RECOMP, B_)  # the compute stream's F/B work (K-FAC items gate on these)
KFAC_STREAM_OPS = (CURV, SYNC_CURV, INV)
_KIND = {WorkKind.Forward: F_, WorkKind.Backward: B_, WorkKind.Recompute: RECOMP, WorkKind.Curvature: CURV,
         WorkKind.SyncCurvature: SYNC_CURV, WorkKind.Inversion: INV, WorkKind.SyncGrad: SYNC_GRAD,
         WorkKind.Precondition: PREC}


@dataclass
class Op:
    kind: str
    stage: int
    step: int
    start: float
    duration: float = 0.0
    micro: Optional[int] = None
    layer: Optional[int] = None
    factor: Optional[int] = None          # 0 = A-set, 1 = B-set
    recv: Optional[Tuple] = None          # channel key (src, dst, pipe, what)
    send: Optional[Tuple] = None
    group: Optional[Tuple[int, ...]] = None  # replica devices of a collective
    gate: Optional[int] = None            # index of the F/B op this K-FAC op waits for
    synthetic: bool = False               # not in the reference timeline (A.8 / A.10)

    def key(self):
        return (self.kind, self.stage, self.micro, self.layer, self.factor, self.step)


@dataclass
class Topology:
    """Stage <-> device mapping of a PipelineConfig (reference schedule.cpp:116,
    bubblefill.cpp:18-41)."""
    cfg: S.PipelineConfig

    @property
    def D(self) -> int:
        return self.cfg.stages

    def pipe_of(self, micro: int) -> int:
        return 1 if (self.cfg.method == Method.Chimera and micro >= self.cfg.micro_batches // 2) else 0

    def device(self, pipe: int, stage: int, group: int) -> int:
        return group * self.D + (stage if pipe == 0 else self.D - 1 - stage)

    def replicas(self, stage: int) -> Tuple[int, ...]:
        """Devices hosting `stage`, in the reference's replica order
        (bubblefill.cpp:18-26): per group g, the down host then the up host."""
        out = []
        for g in range(self.cfg.groups()):
            out.append(self.device(0, stage, g))
            if self.cfg.method == Method.Chimera:
                out.append(self.device(1, stage, g))
        return tuple(out)

    def stages_on(self, dev: int) -> List[int]:
        s = dev % self.D
        return [s, self.D - 1 - s] if self.cfg.method == Method.Chimera else [s]

    def n_devices(self) -> int:
        return self.cfg.effective_devices()


def _channels_for(topo: Topology, dev: int, kind: str, stage: int, micro: int):
    pipe = topo.pipe_of(micro)
    g = dev // topo.D
    recv = send = None
    if kind == F_:
        if stage > 0:
            recv = (topo.device(pipe, stage - 1, g), dev, pipe, "act")
        if stage < topo.D - 1:
            send = (dev, topo.device(pipe, stage + 1, g), pipe, "act")
    elif kind == B_:
        if stage < topo.D - 1:
            recv = (topo.device(pipe, stage + 1, g), dev, pipe, "grad")
        if stage > 0:
            send = (dev, topo.device(pipe, stage - 1, g), pipe, "grad")
    return recv, send


def device_programs(filled: S.FilledSchedule, cfg: S.PipelineConfig,
                    inversion_broadcast: Optional[bool] = None) -> List[List[Op]]:
    """One refresh cycle (filled.refresh_period steps) of ops per device, in
    schedule-time order (ties by the reference's (start, kind) order; a
    SyncGrad precedes the Precondition of its stage — A.6).

    ``inversion_broadcast`` (default: whenever a stage has replicas): the
    reference runs each (layer, factor) Inversion on ONE replica -- the front
    one, or round-robin under inversion parallelism (bubblefill.cpp:162-173,
    :277-285) -- and models no transfer (A.8); every other replica needs the
    inverse, so the runtime broadcasts it from the inverting device."""
    if inversion_broadcast is None:
        inversion_broadcast = cfg.replicas > 1
    topo = Topology(cfg)
    nd = topo.n_devices()
    progs: List[List[Op]] = [[] for _ in range(nd)]
    for dev, line in enumerate(filled.schedule.timelines):
        for w in line:
            kind = _KIND.get(w.kind)
            if kind is None:
                raise ValueError(f"runtime: unsupported work kind {w.kind!r}")
            op = Op(kind, w.stage, w.step, w.start, w.duration, w.micro_batch, w.layer,
                    None if w.factor is None else int(w.factor))
            if kind in (F_, B_):
                op.recv, op.send = _channels_for(topo, dev, kind, w.stage, w.micro_batch)
            if kind in (SYNC_CURV, SYNC_GRAD):
                op.group = topo.replicas(w.stage)
            progs[dev].append(op)
    rank = {k: i for i, k in enumerate((F_, RECOMP, B_, CURV, INV, SYNC_GRAD, PREC, SYNC_CURV))}
    for p in progs:
        # stable: the assigner already sorted by (start, int(kind)); SyncGrad
        # must come before the Precondition of the same stage at equal start
        p.sort(key=lambda o: (o.start, 0 if o.kind == SYNC_GRAD else 1, rank[o.kind]))
    if cfg.replicas > 1:
        _add_curvature_sync_participants(progs, topo)
        if inversion_broadcast:
            _add_inverse_broadcasts(progs, topo)
        _canonicalize_collectives(progs, topo)
    for p in progs:
        _assign_gates(p)
    return progs


def _add_curvature_sync_participants(progs: List[List[Op]], topo: Topology):
    """the reference puts SyncCurvature on devs.front() only; a
    real all-reduce needs every replica.  The other replicas get the same op
    (same schedule time: the front's item starts after every replica's
    curvature of that (layer, factor), reference bubblefill.cpp:150-161);
    _canonicalize_collectives places it."""
    for stage in range(topo.D):
        devs = topo.replicas(stage)
        for s in [o for o in progs[devs[0]] if o.kind == SYNC_CURV and o.stage == stage]:
            for dev in devs[1:]:
                progs[dev].append(Op(SYNC_CURV, stage, s.step, s.start, 0.0, None, s.layer, s.factor,
                                     group=devs, synthetic=True))


def _add_inverse_broadcasts(progs: List[List[Op]], topo: Topology):
    """Inversion parallelism (reference bubblefill.cpp:275-285) only moves the
    Inversion item to another replica; the replicas then need the owner's
    inverse (A.8): every replica joins a broadcast at the item's end time."""
    for stage in range(topo.D):
        devs = topo.replicas(stage)
        for owner in devs:
            for inv in [o for o in progs[owner] if o.kind == INV and o.stage == stage]:
                for dev in devs:
                    progs[dev].append(Op("BCAST_INV", stage, inv.step, inv.start + inv.duration, 0.0, owner,
                                         inv.layer, inv.factor, group=devs, synthetic=True))


_COLL_RANK = {SYNC_CURV: 0, "BCAST_INV": 1, SYNC_GRAD: 2}


def _canonicalize_collectives(progs: List[List[Op]], topo: Topology):
    """All collectives of one replica group go through one communicator, so
    every member must issue them in ONE order.  Canonical order: (schedule
    time, kind, layer, factor, step).  Each member re-inserts them in that
    order, each no earlier than its time slot and its local dependency (the
    device's last curvature of the key for SyncCurvature, the inversion for
    the owner's broadcast) and after the previous collective; a SyncGrad
    still precedes the Precondition of its stage (time ties, A.6)."""
    eps = 1e-9
    for stage in range(topo.D):
        devs = topo.replicas(stage)
        if len(devs) < 2:
            continue
        canon = {}
        for dev in devs:
            for o in progs[dev]:
                if o.group == devs and o.kind in _COLL_RANK:
                    k = (o.kind, o.layer, o.factor, o.step, o.micro)
                    canon.setdefault(k, o.start)
        order = sorted(canon, key=lambda k: (canon[k], _COLL_RANK[k[0]], k[1] if k[1] is not None else -1,
                                             k[2] if k[2] is not None else -1, k[3]))
        for dev in devs:
            mine = {}
            rest = []
            for o in progs[dev]:
                if o.group == devs and o.kind in _COLL_RANK:
                    mine[(o.kind, o.layer, o.factor, o.step, o.micro)] = o
                else:
                    rest.append(o)
            prev = -1
            for k in order:
                o = mine[k]
                t = canon[k]
                pos = next((i for i, q in enumerate(rest) if q.start >= t - eps), len(rest))
                if o.kind == SYNC_CURV:
                    dep = max((i for i, q in enumerate(rest) if q.kind == CURV and q.stage == stage and
                               q.layer == o.layer and q.factor == o.factor and q.step == o.step), default=-1)
                    pos = max(pos, dep + 1)
                elif o.kind == "BCAST_INV" and o.micro == dev:
                    dep = next(i for i, q in enumerate(rest) if q.kind == INV and q.stage == stage and
                               q.layer == o.layer and q.factor == o.factor and q.step == o.step)
                    pos = max(pos, dep + 1)
                pos = max(pos, prev + 1)
                o.start = t
                rest.insert(pos, o)
                prev = pos
            progs[dev][:] = rest


def _assign_gates(p: List[Op]):
    last_fb = None
    for i, o in enumerate(p):
        if o.kind in COMPUTE_OPS:
            last_fb = i
        elif o.kind in KFAC_STREAM_OPS or o.kind == "BCAST_INV":
            o.gate = last_fb


def inline_program(cfg: S.PipelineConfig, refresh: int) -> List[Op]:
    """D = 1, W = 1: no bubbles.  Step k of an R-step cycle: 1F1B order F/B
    (with cfg.recompute, a Recompute of the micro-batch glued in front of its
    Backward, reference schedule.cpp:188-189, :215-223); in step 0 the
    Curvature items of micro-batch m (every layer and set) right after m's
    Backward -- its A and B tapes are complete there, so they run on the
    K-FAC stream beside the remaining F/B instead of after the step (same
    items, same micro-batch order per factor: the same bits); then
    Inversion for every (layer, set), then Precondition."""
    if cfg.stages != 1:
        raise ValueError("inline_program is the single-stage (D = 1) case")
    n, L = cfg.micro_batches, cfg.layers_per_stage
    prog: List[Op] = []
    t = 0.0
    for k in range(refresh):
        fb = [(F_, 0)] + [x for m in range(1, n) for x in ((B_, m - 1), (F_, m))] + [(B_, n - 1)]
        if cfg.recompute:
            fb = [x for kind, m in fb for x in (((RECOMP, m), (B_, m)) if kind == B_ else ((kind, m),))]
        for kind, m in fb:
            prog.append(Op(kind, 0, k, t, 1.0, m))
            t += 1.0
            if k == 0 and kind == B_:
                for l in range(L):
                    for f in (0, 1):
                        prog.append(Op(CURV, 0, k, t, 0.0, m, l, f))
        if k == 0:
            for l in range(L):
                for f in (0, 1):
                    prog.append(Op(INV, 0, k, t, 0.0, None, l, f))
        prog.append(Op(PREC, 0, k, t, 0.0))
    _assign_gates(prog)
    return prog


def channel_plan(progs: Sequence[Sequence[Op]]) -> List[Tuple]:
    """Every P2P channel, in a canonical order (all ranks create the same
    groups in the same order)."""
    chans = set()
    for p in progs:
        for o in p:
            for c in (o.recv, o.send):
                if c is not None:
                    chans.add(c)
    return sorted(chans)


def check_channel_fifo(progs: Sequence[Sequence[Op]]) -> None:
    """Both ends of every channel see the same micro-batch sequence."""
    sends: Dict[Tuple, List] = {}
    recvs: Dict[Tuple, List] = {}
    for p in progs:
        for o in p:
            if o.send is not None:
                sends.setdefault(o.send, []).append((o.step, o.micro))
            if o.recv is not None:
                recvs.setdefault(o.recv, []).append((o.step, o.micro))
    if sends.keys() != recvs.keys():
        raise AssertionError("unpaired channel")
    for c in sends:
        if sends[c] != recvs[c]:
            raise AssertionError(f"channel {c}: send order {sends[c]} != recv order {recvs[c]}")


def check_collective_order(progs: Sequence[Sequence[Op]]) -> None:
    """Every member of a replica group issues its collectives in one order."""
    seqs: Dict[Tuple, Dict[int, List]] = {}
    for dev, p in enumerate(progs):
        for o in p:
            if o.group is not None and o.kind in (SYNC_CURV, SYNC_GRAD, "BCAST_INV"):
                seqs.setdefault(o.group, {}).setdefault(dev, []).append((o.kind, o.stage, o.layer, o.factor, o.step))
    for g, per in seqs.items():
        orders = list(per.values())
        if any(x != orders[0] for x in orders) or set(per) != set(g):
            raise AssertionError(f"collective order differs within group {g}: {per}")


# ---------------------------------------------------------------------- execution
@dataclass
class StepStats:
    step_ms: float = 0.0
    busy_ms: float = 0.0
    util: float = 0.0
    loss: float = 0.0
    ops: List[Tuple[str, float, float]] = field(default_factory=list)  # (kind, begin_ms, end_ms)


class Executor:
    """Runs a device program with a pluggable backend.

    The backend supplies the arithmetic: ``CudaBackend`` (product: BERT F/B
    in torch, K-FAC through libpf_b200.so) or a test double in the CPU
    tests.  Communication goes through ``comm`` (torch.distributed groups).
    """

    def __init__(self, program: List[Op], backend, comm, rank: int):
        self.program, self.backend, self.comm, self.rank = program, backend, comm, rank

    def run_cycle(self, cycle: int) -> None:
        b, comm = self.backend, self.comm
        fb_done: Dict[int, object] = {}
        prog = self.program
        i = 0
        while i < len(prog):
            op = prog[i]
            b.cur_step, b.cur_op, b.cur_gate = op.step, i, op.gate  # trace metadata
            # a run of consecutive Curvature / Inversion items behind the same
            # gate becomes ONE backend call (one grouped SYRK launch / one
            # batched inverse whose independent chains overlap)
            if op.kind in (CURV, INV) and hasattr(b, "curvature_many"):
                j = i
                while j < len(prog) and prog[j].kind == op.kind and prog[j].gate == op.gate:
                    j += 1
                gate = fb_done.get(op.gate) if op.gate is not None else None
                items = [(o.stage, o.layer, o.factor, o.micro) for o in prog[i:j]]
                if op.kind == CURV:
                    b.curvature_many(items, gate)
                else:
                    b.invert_many([it[:3] for it in items], gate)
                i = j
                continue
            i += 1
            if op.kind == F_:
                x = comm.recv(op.recv, b.act_shape(op.stage, op.micro)) if op.recv else None
                y = b.forward(op.stage, op.micro, x, capture=(op.step == 0), cycle=cycle)
                if op.send:
                    comm.send(op.send, y)
                fb_done[i - 1] = b.mark_compute()
            elif op.kind == RECOMP:
                # activation recomputation (reference WorkKind::Recompute): the
                # forward of this micro-batch again, from its saved stage input,
                # right before its backward on the same device
                b.recompute(op.stage, op.micro)
                fb_done[i - 1] = b.mark_compute()
            elif op.kind == B_:
                gy = comm.recv(op.recv, b.act_shape(op.stage, op.micro)) if op.recv else None
                gx = b.backward(op.stage, op.micro, gy, capture=(op.step == 0))
                if op.send:
                    comm.send(op.send, gx)
                fb_done[i - 1] = b.mark_compute()
            else:
                gate = fb_done.get(op.gate) if op.gate is not None else None
                if op.kind == CURV:
                    b.curvature(op.stage, op.layer, op.factor, op.micro, gate)
                elif op.kind == SYNC_CURV:
                    b.sync_curvature(op.stage, op.layer, op.factor, comm.group(op.group), gate)
                elif op.kind == INV:
                    b.invert(op.stage, op.layer, op.factor, gate)
                elif op.kind == "BCAST_INV":
                    b.broadcast_inverse(op.stage, op.layer, op.factor, op.micro, comm.group(op.group), gate)
                elif op.kind == SYNC_GRAD:
                    b.sync_grad(op.stage, comm.group(op.group))
                elif op.kind == PREC:
                    b.precondition(op.stage, op.step)
                else:  # pragma: no cover
                    raise ValueError(op.kind)
        b.end_cycle()


class Comm:
    """torch.distributed plumbing: one 2-rank group per P2P channel, one group
    per replica set, created in a canonical order on every rank."""

    def __init__(self, dist, rank: int, channels: Sequence[Tuple], replica_sets: Sequence[Tuple[int, ...]],
                 device=None):
        self.dist, self.rank, self.device = dist, rank, device
        self.chan_groups = {}
        for c in channels:
            g = dist.new_group(sorted({c[0], c[1]}))
            self.chan_groups[c] = g
        self.groups = {}
        for rs in sorted(set(tuple(r) for r in replica_sets)):
            self.groups[rs] = dist.new_group(list(rs)) if len(rs) > 1 else None
        self.pending: List = []

    def group(self, devs):
        return self.groups.get(tuple(devs))

    def send(self, chan, tensor):
        assert chan[0] == self.rank
        t = tensor.contiguous()
        self.pending.append((self.dist.isend(t, chan[1], group=self.chan_groups[chan]), t))

    def recv(self, chan, shape_dtype):
        assert chan[1] == self.rank
        shape, dtype = shape_dtype
        import torch
        buf = torch.empty(shape, dtype=dtype, device=self.device)
        self.dist.irecv(buf, chan[0], group=self.chan_groups[chan]).wait()
        return buf

    def flush(self):
        for w, _ in self.pending:
            w.wait()
        self.pending.clear()
