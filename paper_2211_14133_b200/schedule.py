"""Python mirror of the reference scheduler API (``pipefill::`` in
/root/reference/proj/include/pipefill/{core,schedule,bubblefill}.hpp), backed
by the C-ABI (include/pf_sched.h) of the C++ host scheduler in
``csrc/host/{schedule,bubblefill}.cpp``.

Names, fields, defaults and error behaviour follow the reference:
``build_schedule`` raises ``ValueError`` (std::invalid_argument),
``assign_works`` raises :class:`InfeasibleError` carrying ``unplaced`` and
``deficit_ms`` (bubblefill.hpp:56-65).
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import List, Optional

from . import _lib as L


class Method(enum.IntEnum):
    GPipe = 0
    OneF1B = 1
    Chimera = 2


class Factor(enum.IntEnum):
    A = 0
    B = 1


class WorkKind(enum.IntEnum):
    Forward = 0
    Backward = 1
    Recompute = 2
    Curvature = 3
    Inversion = 4
    Precondition = 5
    SyncGrad = 6
    SyncCurvature = 7


_KIND_NAMES = ["forward", "backward", "recompute", "curvature", "inversion", "precondition",
               "sync-grad", "sync-curvature"]


def kind_name(k: WorkKind) -> str:
    return _KIND_NAMES[int(k)]


def parse_method(name: str) -> Optional[Method]:
    return {"gpipe": Method.GPipe, "1f1b": Method.OneF1B, "onef1b": Method.OneF1B,
            "chimera": Method.Chimera}.get(name)


@dataclass
class PipelineConfig:  # core.hpp:35-61
    method: Method = Method.GPipe
    stages: int = 1
    micro_batches: int = 1
    micro_batch_size: int = 1
    replicas: int = 1
    devices: int = 0
    layers_per_stage: int = 1
    seq_len: int = 128
    recompute: bool = False

    def stages_per_device(self) -> int:
        return 2 if self.method == Method.Chimera else 1

    def effective_devices(self) -> int:
        return self.devices if self.devices > 0 else \
            self.stages * self.replicas // self.stages_per_device()

    def groups(self) -> int:
        return self.replicas // self.stages_per_device()

    def mini_batch_size(self) -> int:
        return self.micro_batch_size * self.micro_batches * self.replicas

    def _c(self) -> L.PfConfig:
        return L.PfConfig(int(self.method), self.stages, self.micro_batches,
                          self.micro_batch_size, self.replicas, self.devices,
                          self.layers_per_stage, self.seq_len, int(bool(self.recompute)))


@dataclass
class CostTable:  # core.hpp:67-87
    t_f: float = 0.0
    t_b: float = 0.0
    t_curv: float = 0.0
    t_inv: float = 0.0
    t_prec: float = 0.0
    m_theta: int = 0
    m_act: int = 0
    m_err_peak: int = 0
    m_err_save: int = 0
    m_curv: int = 0
    comm_alpha: float = 0.0
    comm_beta: float = math.inf
    p2p_latency: float = 0.0

    def m_inv(self) -> int:
        return self.m_curv

    def _c(self) -> L.PfCosts:
        return L.PfCosts(self.t_f, self.t_b, self.t_curv, self.t_inv, self.t_prec, self.m_theta,
                         self.m_act, self.m_err_peak, self.m_err_save, self.m_curv,
                         self.comm_alpha, self.comm_beta, self.p2p_latency)


@dataclass
class WorkItem:  # core.hpp:89-102
    kind: WorkKind = WorkKind.Forward
    stage: int = -1
    micro_batch: Optional[int] = None
    layer: Optional[int] = None
    factor: Optional[Factor] = None
    device: int = -1
    start: float = 0.0
    duration: float = 0.0
    step: int = 0

    def end(self) -> float:
        return self.start + self.duration


@dataclass
class Interval:
    begin: float = 0.0
    end: float = 0.0

    def length(self) -> float:
        return self.end - self.begin


@dataclass
class StalenessEntry:
    stage: int = 0
    layer: int = 0
    staleness_steps: int = 0


@dataclass
class StaticSchedule:  # core.hpp:106-115
    timelines: List[List[WorkItem]] = field(default_factory=list)
    period: float = 0.0
    horizon_steps: int = 1
    refresh_period: int = 1
    _handle: Optional["_Handle"] = field(default=None, repr=False, compare=False)

    def device_count(self) -> int:
        return len(self.timelines)

    def makespan(self) -> float:
        return max((w.end() for line in self.timelines for w in line), default=0.0)


@dataclass
class FilledSchedule:  # bubblefill.hpp:46-54
    schedule: StaticSchedule
    base_period: float = 0.0
    refresh_period: int = 1
    staleness: List[StalenessEntry] = field(default_factory=list)
    preconditions_using_prior_inverses: int = 0


@dataclass
class KfacWork:  # bubblefill.hpp:16-29
    kind: WorkKind = WorkKind.Curvature
    stage: int = 0
    layer: int = 0
    factor: Factor = Factor.A
    micro_batch: Optional[int] = None
    device: int = 0
    duration: float = 0.0
    base_anchor: Optional[WorkKind] = None
    preds: List[int] = field(default_factory=list)


@dataclass
class KfacWorkQueue:
    items: List[KfacWork] = field(default_factory=list)


@dataclass
class AssignOptions:
    inversion_parallel: bool = False
    horizon_cap: int = 10


class InfeasibleError(RuntimeError):  # bubblefill.hpp:56-65
    def __init__(self, message: str, unplaced: List[KfacWork], deficit_ms: float):
        super().__init__(message)
        self.unplaced = unplaced
        self.deficit_ms = deficit_ms


class _Handle:
    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            L.lib().pf_schedule_free(self.ptr)
            self.ptr = 0


def _opt(v: int) -> Optional[int]:
    return None if v < 0 else int(v)


def _item(c: L.PfItem) -> WorkItem:
    return WorkItem(WorkKind(c.kind), c.stage, _opt(c.micro_batch), _opt(c.layer),
                    None if c.factor < 0 else Factor(c.factor), c.device, c.start, c.duration,
                    c.step)


def _work(c: L.PfWork, preds: List[int]) -> KfacWork:
    return KfacWork(WorkKind(c.kind), c.stage, c.layer, Factor(c.factor), _opt(c.micro_batch),
                    c.device, c.duration, None if c.base_anchor < 0 else WorkKind(c.base_anchor),
                    preds)


def _materialize(ptr: int) -> StaticSchedule:
    lib = L.lib()
    devices, horizon, refresh, prior = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    period, base_period, span = C.c_double(), C.c_double(), C.c_double()
    L.check(lib.pf_schedule_info(ptr, devices, period, horizon, refresh, base_period, prior, span),
            "pf_schedule_info")
    timelines = []
    for d in range(devices.value):
        n = C.c_int()
        L.check(lib.pf_schedule_timeline(ptr, d, None, 0, n), "pf_schedule_timeline")
        buf = (L.PfItem * max(1, n.value))()
        L.check(lib.pf_schedule_timeline(ptr, d, buf, n.value, n), "pf_schedule_timeline")
        timelines.append([_item(buf[i]) for i in range(n.value)])
    return StaticSchedule(timelines, period.value, horizon.value, refresh.value, _Handle(ptr))


def validate_config(config: PipelineConfig) -> List[tuple]:
    buf = C.create_string_buffer(8192)
    n = C.c_int()
    L.check(L.lib().pf_validate_config(config._c(), buf, len(buf), n), "validate_config")
    if n.value == 0:
        return []
    return [tuple(line.split(": ", 1)) for line in buf.value.decode().split("\n")]


def build_schedule(config: PipelineConfig, costs: CostTable, horizon_steps: int = 1) -> StaticSchedule:
    """schedule.hpp:29-30."""
    out = C.c_void_p()
    L.check(L.lib().pf_build_schedule(config._c(), costs._c(), horizon_steps, out),
            "build_schedule")
    return _materialize(out.value)


def extract_bubbles(schedule: StaticSchedule):
    """schedule.hpp:34 — returns (idle per device, total idle per device)."""
    _require_handle(schedule)
    lib = L.lib()
    idle, totals = [], []
    for d in range(schedule.device_count()):
        n, tot = C.c_int(), C.c_double()
        L.check(lib.pf_extract_bubbles(schedule._handle.ptr, d, None, 0, n, tot), "extract_bubbles")
        buf = (L.PfInterval * max(1, n.value))()
        L.check(lib.pf_extract_bubbles(schedule._handle.ptr, d, buf, n.value, n, tot),
                "extract_bubbles")
        idle.append([Interval(buf[i].begin, buf[i].end) for i in range(n.value)])
        totals.append(tot.value)
    return idle, totals


def schedule_metrics(schedule: StaticSchedule):
    """schedule.hpp:42 — (makespan, utilization, per_device_busy)."""
    _require_handle(schedule)
    span, util = C.c_double(), C.c_double()
    busy = (C.c_double * max(1, schedule.device_count()))()
    L.check(L.lib().pf_schedule_metrics(schedule._handle.ptr, span, util, busy), "schedule_metrics")
    return span.value, util.value, list(busy)[: schedule.device_count()]


def validate_schedule(schedule: StaticSchedule, config: PipelineConfig) -> List[tuple]:
    _require_handle(schedule)
    buf = C.create_string_buffer(1 << 20)
    n = C.c_int()
    L.check(L.lib().pf_validate_schedule(schedule._handle.ptr, config._c(), buf, len(buf), n),
            "validate_schedule")
    if n.value == 0:
        return []
    return [tuple(line.split(": ", 1)) for line in buf.value.decode().split("\n")]


def model_collective(bytes_: float, participants: int, alpha: float, beta: float) -> float:
    out = C.c_double()
    L.check(L.lib().pf_model_collective(bytes_, participants, alpha, beta, out), "model_collective")
    return out.value


class _Queue:
    def __init__(self, ptr: int):
        self.ptr = ptr

    def __del__(self):
        if self.ptr:
            L.lib().pf_queue_free(self.ptr)


def _queue_items(ptr: int) -> List[KfacWork]:
    lib = L.lib()
    n = C.c_int()
    L.check(lib.pf_queue_size(ptr, n), "queue")
    out = []
    for i in range(n.value):
        w = L.PfWork()
        L.check(lib.pf_queue_get(ptr, i, w, None, 0), "queue")
        preds = (C.c_int32 * max(1, w.n_preds))()
        L.check(lib.pf_queue_get(ptr, i, w, preds, w.n_preds), "queue")
        out.append(_work(w, list(preds)[: w.n_preds]))
    return out


def enumerate_kfac_works(config: PipelineConfig, costs: CostTable) -> KfacWorkQueue:
    """bubblefill.hpp:71."""
    out = C.c_void_p()
    L.check(L.lib().pf_enumerate_kfac_works(config._c(), costs._c(), out), "enumerate_kfac_works")
    q = _Queue(out.value)
    return KfacWorkQueue(_queue_items(q.ptr))


def _push_queue(queue: KfacWorkQueue) -> _Queue:
    lib = L.lib()
    q = _Queue(lib.pf_queue_new())
    for w in queue.items:
        c = L.PfWork(int(w.kind), w.stage, w.layer, int(w.factor),
                     -1 if w.micro_batch is None else w.micro_batch, w.device, w.duration,
                     -1 if w.base_anchor is None else int(w.base_anchor), len(w.preds))
        preds = (C.c_int32 * max(1, len(w.preds)))(*w.preds)
        L.check(lib.pf_queue_push(q.ptr, c, preds), "queue push")
    return q


def _require_handle(s: StaticSchedule):
    if s._handle is None:
        raise ValueError("schedule was not produced by build_schedule/assign_works")


def assign_works(base: StaticSchedule, config: PipelineConfig, costs: CostTable,
                 queue: KfacWorkQueue, opts: AssignOptions = AssignOptions()) -> FilledSchedule:
    """bubblefill.hpp:83-85."""
    _require_handle(base)
    lib = L.lib()
    q = _push_queue(queue)
    out = C.c_void_p()
    rc = lib.pf_assign_works(base._handle.ptr, config._c(), costs._c(), q.ptr,
                             int(opts.inversion_parallel), opts.horizon_cap, out)
    if rc == L.PF_INFEASIBLE:
        h = _Handle(out.value)
        msg = lib.pf_last_error().decode()
        deficit, n = C.c_double(), C.c_int()
        L.check(lib.pf_infeasible_payload(h.ptr, deficit, n), "infeasible payload")
        unplaced = []
        for i in range(n.value):
            w = L.PfWork()
            L.check(lib.pf_infeasible_item(h.ptr, i, w), "infeasible item")
            unplaced.append(_work(w, []))
        raise InfeasibleError(msg, unplaced, deficit.value)
    L.check(rc, "assign_works")
    sched = _materialize(out.value)
    info_prior = C.c_int()
    base_period = C.c_double()
    L.check(lib.pf_schedule_info(out.value, None, None, None, None, base_period, info_prior, None),
            "info")
    n = C.c_int()
    L.check(lib.pf_schedule_staleness(out.value, None, 0, n), "staleness")
    buf = (L.PfStaleness * max(1, n.value))()
    L.check(lib.pf_schedule_staleness(out.value, buf, n.value, n), "staleness")
    stale = [StalenessEntry(buf[i].stage, buf[i].layer, buf[i].staleness_steps)
             for i in range(n.value)]
    return FilledSchedule(sched, base_period.value, sched.refresh_period, stale, info_prior.value)


def staleness_report(filled: FilledSchedule) -> List[StalenessEntry]:
    _require_handle(filled.schedule)
    n = C.c_int()
    L.check(L.lib().pf_staleness_report(filled.schedule._handle.ptr, None, 0, n), "staleness")
    buf = (L.PfStaleness * max(1, n.value))()
    L.check(L.lib().pf_staleness_report(filled.schedule._handle.ptr, buf, n.value, n), "staleness")
    return [StalenessEntry(buf[i].stage, buf[i].layer, buf[i].staleness_steps)
            for i in range(n.value)]
