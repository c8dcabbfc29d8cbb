"""PipeFisher trainer: BERT stages + K-FAC state + the runtime (runtime.py).

``CudaBackend`` is the product backend: F/B of the hosted BERT stages on the
compute stream (torch / cuBLAS — the bubble-creating work), every K-FAC
operation through libpf_b200.so (kfac.py): grouped tcgen05 SYRK curvature,
batched fp32-accurate damped inverses written in digit form, and the grouped
fused precondition-update.  Nothing here has a CPU path.

Per hosted stage and encoder layer the factor sets are:
  A-set: a_qkv (Q/K/V share one input), a_o, a_ffn1, a_ffn2   -> 4 factors
  B-set: e_q, e_k, e_v, e_o, e_ffn1, e_ffn2                    -> 6 factors
"""
from __future__ import annotations

import os

import math
import time
from dataclasses import dataclass
from typing import Dict, List, Optional, Tuple

import torch

from . import kfac as K
from . import runtime as R
from . import schedule as S
from .bert import BertConfig, BertStage, synthetic_batch

A_KEYS = ("a_qkv", "a_o", "a_ffn1", "a_ffn2")
E_KEYS = ("e_q", "e_k", "e_v", "e_o", "e_ffn1", "e_ffn2")
LINEAR_FACTORS = {"q": ("a_qkv", "e_q"), "k": ("a_qkv", "e_k"), "v": ("a_qkv", "e_v"),
                  "o": ("a_o", "e_o"), "ffn1": ("a_ffn1", "e_ffn1"), "ffn2": ("a_ffn2", "e_ffn2")}


def factor_dim(bert: BertConfig, key: str) -> int:
    return bert.ffn if key in ("a_ffn2", "e_ffn1") else bert.hidden


class StageKfac:
    """Factors, double-buffered inverses (fp32 + digit form) and the
    per-cycle accumulation state of one hosted stage."""

    def __init__(self, bert: BertConfig, layers: int, device):
        self.bert, self.layers = bert, layers
        self.factor: Dict[Tuple[int, str], torch.Tensor] = {}
        self.inv: Dict[Tuple[int, str, int], K.SlicedMatrix] = {}
        for l in range(layers):
            for key in A_KEYS + E_KEYS:
                d = factor_dim(bert, key)
                self.factor[(l, key)] = torch.zeros((d, d), dtype=torch.float32, device=device)
                for slot in (0, 1):
                    self.inv[(l, key, slot)] = K.SlicedMatrix(
                        torch.zeros((d, d), dtype=torch.float32, device=device),
                        torch.zeros(K.slice_bytes(d, d), dtype=torch.uint8, device=device))
        self.version = {(l, f): -1 for l in range(layers) for f in (0, 1)}  # -1: no inverse yet
        self.started = {(l, f): False for l in range(layers) for f in (0, 1)}
        self.slot_free: Dict[Tuple[int, int, int], Optional[torch.cuda.Event]] = {}
        self.inv_ready: Optional[torch.cuda.Event] = None

    @staticmethod
    def keys(f: int):
        return A_KEYS if f == 0 else E_KEYS


_TRIL: Dict[Tuple[int, str], torch.Tensor] = {}


def _tril_index(d: int, device) -> torch.Tensor:
    """Flat row-major indices of the lower triangle of a d x d matrix (cached)."""
    key = (d, str(device))
    if key not in _TRIL:
        r, c = torch.tril_indices(d, d, device=device)
        _TRIL[key] = r * d + c
    return _TRIL[key]


class _StageCall(torch.nn.Module):
    """One graphed F/B key of a stage (the stage module is shared)."""

    def __init__(self, stage: torch.nn.Module):
        super().__init__()
        self.stage = stage

    def forward(self, x, mlm_positions, mlm_labels):
        return self.stage(x, mlm_positions, mlm_labels)


class CudaBackend:
    def __init__(self, topo: R.Topology, bert: BertConfig, rank: int, device, kfac: bool = True,
                 damping: float = 0.1, lr: float = 1e-3, seed: int = 0, dist=None, graph_fb: bool = False):
        cfg = topo.cfg
        if dist is None:
            import torch.distributed as dist
        self.dist = dist  # torch.distributed, or the in-process stand-in of vdev.py
        self.topo, self.bert, self.rank, self.device, self.use_kfac = topo, bert, rank, device, kfac
        self.damping, self.lr = damping, lr
        self.B, self.Sq, L = cfg.micro_batch_size, cfg.seq_len, cfg.layers_per_stage
        self.tokens = self.B * self.Sq
        low, high = torch.cuda.Stream.priority_range()
        # F/B (and the tail) on a high-priority stream made current for torch;
        # K-FAC items on a low-priority stream: when both have CTAs pending the
        # block scheduler serves F/B first
        self.compute = torch.cuda.Stream(device=device, priority=high)
        torch.cuda.set_stream(self.compute)
        self.kfac_stream = torch.cuda.Stream(device=device, priority=low)
        torch.manual_seed(seed + 1000 * rank)
        self.stages: Dict[int, BertStage] = {}
        self.kstate: Dict[int, StageKfac] = {}
        for s in topo.stages_on(rank):
            torch.manual_seed(seed + s)  # replicas of a stage start identical
            st = BertStage(bert, s * L, L, s == 0, s == topo.D - 1).to(device)
            self.stages[s] = st
            if kfac:
                self.kstate[s] = StageKfac(bert, L, device)
        # micro-batches this device runs (its pipe's half under Chimera)
        self.local_micros = {s: sum(1 for m in range(cfg.micro_batches)
                                    if topo.device(topo.pipe_of(m), s, rank // topo.D) == rank)
                             for s in self.stages}
        self.data = {m: synthetic_batch(bert, self.B, self.Sq, seed + 7919 * (rank // topo.D) + m, device)
                     for m in range(cfg.micro_batches)}
        self.saved: Dict[Tuple[int, int], Tuple] = {}
        self.losses: List[torch.Tensor] = []
        self.timeline: List[Tuple[str, torch.cuda.Event, torch.cuda.Event, dict]] = []
        self.record = False
        self.recompute_on = bool(cfg.recompute)  # WorkKind::Recompute items in the program
        # F/B of each (stage, micro-batch, tape capture) as CUDA graphs
        # (torch.cuda.make_graphed_callables): the eager BERT F/B is host-bound
        # (CUPTI kernel utilisation ~0.65 at D = 1).  One graph pair per key, so
        # the step-0 tapes (views of graph-static activations / gradients) stay
        # valid until that key replays in the next refresh cycle, after the
        # cycle-end join with the K-FAC stream.
        self.graph_fb = bool(graph_fb) and not self.recompute_on
        self.graphed: Dict[Tuple[int, int, bool], object] = {}
        self.inv_graphs: Dict[Tuple[int, ...], torch.cuda.CUDAGraph] = {}  # batched inversions (graph_fb)
        self.cur_step = 0  # set by the executor before each op (trace metadata):
        self.cur_op = None  # program index of the op (first of a batched run)
        self.cur_gate = None  # program index of the F/B op it is gated on

    # ------------------------------------------------------------ timing helpers
    def _begin(self, stream):
        if not self.record:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    def _end(self, kind, e0, stream, **meta):
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(stream)
        meta.setdefault("step", self.cur_step)
        meta.setdefault("op", self.cur_op)
        meta.setdefault("gate", self.cur_gate)
        self.timeline.append((kind, e0, e1, meta))

    def mark_compute(self):
        ev = torch.cuda.Event()
        ev.record(self.compute)
        return ev

    def act_shape(self, stage, micro):
        return (self.B, self.Sq, self.bert.hidden), torch.bfloat16

    # ------------------------------------------------------------ F / B
    def forward(self, stage, micro, x, capture, cycle):
        mod = self.stages[stage]
        e0 = self._begin(self.compute)
        ids, pos, labels = self.data[micro]
        if mod.is_first:
            inp = ids
        else:
            inp = x.requires_grad_()
        mod.store.active_micro = micro if (capture and self.use_kfac) else None
        if self.graph_fb:
            key = (stage, micro, bool(capture and self.use_kfac))
            fn = self.graphed.get(key)
            if fn is None:
                # warm-up + capture run the forward / backward on sample inputs
                # (tapes recorded during the capture are the graph's static
                # tensors); parameters' .grad are untouched by the capture
                sample = inp.detach().clone().requires_grad_(not mod.is_first) if not mod.is_first else inp
                # a wrapper per key: make_graphed_callables replaces the forward
                # of the module it is given (its parameters are the stage's)
                fn = torch.cuda.make_graphed_callables(_StageCall(mod), (sample, pos, labels),
                                                       allow_unused_input=True)
                # the capture recorded this key's tapes (forward AND backward):
                # graph-static tensors, re-registered at every replay
                tapes = {k: v for k, v in mod.store.tapes.items() if key[2] and k[2] == micro}
                self.graphed[key] = (fn, tapes)
            fn, tapes = self.graphed[key]
            mod.store.tapes.update(tapes)
            out = fn(inp, pos, labels)
            self.saved[(stage, micro)] = (inp, out)
        elif self.recompute_on:
            # activation recomputation: no autograd graph is kept between F and
            # B, only the stage input; the Recompute op rebuilds it
            with torch.no_grad():
                out = mod(inp.detach() if not mod.is_first else inp, pos, labels)
            self.saved[(stage, micro)] = (inp.detach() if not mod.is_first else inp, None)
        else:
            out = mod(inp, pos, labels)
            self.saved[(stage, micro)] = (inp, out)
        mod.store.active_micro = None
        self._end("F", e0, self.compute, stage=stage, micro_batch=micro)
        if mod.is_last:
            self.losses.append(out.detach())
            return None
        return out.detach().to(torch.bfloat16)

    def recompute(self, stage, micro):
        """WorkKind::Recompute: the micro-batch's forward again from its saved
        stage input, now with autograd (the tapes were captured by the first
        forward; this pass records none)."""
        mod = self.stages[stage]
        e0 = self._begin(self.compute)
        ids, pos, labels = self.data[micro]
        inp, _ = self.saved[(stage, micro)]
        if not mod.is_first:
            inp = inp.requires_grad_()
        mod.store.active_micro = None
        out = mod(inp, pos, labels)
        self.saved[(stage, micro)] = (inp, out)
        self._end("RECOMP", e0, self.compute, stage=stage, micro_batch=micro)

    def backward(self, stage, micro, gy, capture):
        mod = self.stages[stage]
        e0 = self._begin(self.compute)
        inp, out = self.saved.pop((stage, micro))
        mod.store.active_micro = micro if (capture and self.use_kfac) else None
        if mod.is_last:
            (out / self.local_micros[stage]).backward()
        else:
            out.backward(gy.to(out.dtype))
        mod.store.active_micro = None
        self._end("B", e0, self.compute, stage=stage, micro_batch=micro)
        return None if mod.is_first else inp.grad.to(torch.bfloat16)

    # ------------------------------------------------------------ K-FAC items
    def curvature(self, stage, layer, f, micro, gate):
        self.curvature_many([(stage, layer, f, micro)], gate)

    def curvature_many(self, items, gate):
        """Curvature work items -> SYRK problems, one grouped tcgen05 launch.
        The first item of a (layer, set) in a cycle overwrites the factor, the
        others accumulate (the cycle's factor averages its micro-batches)."""
        with torch.cuda.stream(self.kfac_stream):
            if gate is not None:
                self.kfac_stream.wait_event(gate)
            e0 = self._begin(self.kfac_stream)
            probs, pending = [], set()
            for stage, layer, f, micro in items:
                ks, mod = self.kstate[stage], self.stages[stage]
                scale = 1.0 / (self.local_micros[stage] * self.tokens)
                if any((stage, layer, key) in pending for key in ks.keys(f)):
                    # tiles of one launch are unordered: a factor appears at most
                    # once per launch (later micro-batches go to the next launch)
                    K.syrk(probs, fill_upper=False)
                    probs, pending = [], set()
                for key in ks.keys(f):
                    x = mod.store.get(layer, key, micro)
                    x.record_stream(self.kfac_stream)
                    probs.append((x, ks.factor[(layer, key)], scale, ks.started[(layer, f)], True))  # token-major
                    pending.add((stage, layer, key))
                ks.started[(layer, f)] = True
            if probs:
                K.syrk(probs, fill_upper=False)
            st0, l0, f0, m0 = items[0]
            self._end("CURV", e0, self.kfac_stream, stage=st0, layer=l0, factor=f0, micro_batch=m0, items=len(items))

    def sync_curvature(self, stage, layer, f, group, gate):
        """SyncCurvature (bubblefill.cpp:150-161): the replica average of one
        layer's factor set.  The factors are lower-triangular (the SYRK writes
        only the lower tiles), so only the packed lower triangles travel -- all
        of the set's factors in ONE all-reduce of sum d(d+1)/2 floats, the
        m_curv / 2 message the reference's cost model charges."""
        ks = self.kstate[stage]
        with torch.cuda.stream(self.kfac_stream):
            if gate is not None:
                self.kfac_stream.wait_event(gate)
            e0 = self._begin(self.kfac_stream)
            if group is not None:
                mats = [ks.factor[(layer, key)] for key in ks.keys(f)]
                idx = [_tril_index(m.shape[0], m.device) for m in mats]
                packed = torch.cat([m.view(-1).index_select(0, i) for m, i in zip(mats, idx)])
                self.dist.all_reduce(packed, op=self.dist.ReduceOp.AVG, group=group)
                off = 0
                for m, i in zip(mats, idx):
                    m.view(-1).index_copy_(0, i, packed[off:off + i.numel()])
                    off += i.numel()
            self._end("SYNC_CURV", e0, self.kfac_stream, stage=stage, layer=layer, factor=f)

    def invert(self, stage, layer, f, gate):
        self.invert_many([(stage, layer, f)], gate)

    def invert_many(self, items, gate):
        """Inversion work items -> ONE batched damped-inverse call (equal-d
        factors share launches, independent chains overlap on side streams),
        into the free slot of each double-buffered inverse."""
        mats, outs, digs = [], [], []
        with torch.cuda.stream(self.kfac_stream):
            if gate is not None:
                self.kfac_stream.wait_event(gate)
            for stage, layer, f in items:
                ks = self.kstate[stage]
                slot = (ks.version[(layer, f)] + 1) % 2
                free = ks.slot_free.get((layer, f, slot))
                if free is not None:  # last precondition that read this slot
                    self.kfac_stream.wait_event(free)
                for k in ks.keys(f):
                    mats.append(ks.factor[(layer, k)])
                    o = ks.inv[(layer, k, slot)]
                    outs.append(o.fp32)
                    digs.append(o.digits)
            e0 = self._begin(self.kfac_stream)
            if self.graph_fb:
                # a batched inversion is thousands of dependent launches: the
                # first call with a set of buffers runs eagerly (library
                # warm-up) and is then captured as a CUDA graph that every
                # later call replays (24-layer batch: 47 -> ~27 ms, host-bound
                # when issued eagerly)
                key = tuple(t.data_ptr() for t in mats + outs + digs)
                g = self.inv_graphs.get(key)
                if g is not None:
                    g.replay()
                else:
                    K.damped_inverse_batched(mats, self.damping, outs, digs, check=False)
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.kfac_stream):
                        K.damped_inverse_batched(mats, self.damping, outs, digs, check=False)
                    self.inv_graphs[key] = g
            else:
                K.damped_inverse_batched(mats, self.damping, outs, digs, check=False)
            st0, l0, f0 = items[0]
            self._end("INV", e0, self.kfac_stream, stage=st0, layer=l0, factor=f0, items=len(items))
            ev = torch.cuda.Event()
            ev.record(self.kfac_stream)
        for stage, layer, f in items:
            ks = self.kstate[stage]
            ks.version[(layer, f)] += 1
            ks.started[(layer, f)] = False
            ks.inv_ready = ev

    def broadcast_inverse(self, stage, layer, f, owner, group, gate):
        ks = self.kstate[stage]
        dist = self.dist
        if owner != self.rank:
            ks.version[(layer, f)] += 1
            ks.started[(layer, f)] = False  # the next cycle's curvature starts a fresh factor here too
        slot = ks.version[(layer, f)] % 2
        with torch.cuda.stream(self.kfac_stream):
            if gate is not None:
                self.kfac_stream.wait_event(gate)
            free = ks.slot_free.get((layer, f, slot))
            if free is not None:  # the last precondition that read this slot's older version
                self.kfac_stream.wait_event(free)
            for key in ks.keys(f):
                # the preconditioner consumes only the digit form; the fp32
                # inverse stays on the owner (non-owners never read it)
                m = ks.inv[(layer, key, slot)]
                dist.broadcast(m.digits, src=owner, group=group)
            ev = torch.cuda.Event()
            ev.record(self.kfac_stream)
        ks.inv_ready = ev

    def sync_grad(self, stage, group):
        if group is None:
            return
        dist = self.dist
        e0 = self._begin(self.compute)
        grads = [p.grad for p in self.stages[stage].parameters() if p.grad is not None]
        flat = torch.cat([g.reshape(-1) for g in grads])
        dist.all_reduce(flat, op=dist.ReduceOp.AVG, group=group)
        off = 0
        for g in grads:
            g.copy_(flat[off:off + g.numel()].view_as(g))
            off += g.numel()
        self._end("SYNC_GRAD", e0, self.compute, stage=stage)

    def precondition(self, stage, step):
        mod = self.stages[stage]
        e0 = self._begin(self.compute)
        kfac_params = set()
        if self.use_kfac:
            ks = self.kstate[stage]
            if ks.inv_ready is not None:
                self.compute.wait_event(ks.inv_ready)
                ks.inv_ready = None
            items = []
            for l, layer in enumerate(mod.kfac_layers()):
                va, vb = ks.version[(l, 0)], ks.version[(l, 1)]
                for name, (ak, ek) in LINEAR_FACTORS.items():
                    w = layer.w[name]
                    kfac_params.add(id(w))
                    if w.grad is None:
                        continue
                    if va < 0 or vb < 0:  # no inverse yet: the plain gradient (A.13)
                        w.data.add_(w.grad, alpha=-self.lr)
                        continue
                    items.append((w.data, w.grad, ks.inv[(l, ak, va % 2)], ks.inv[(l, ek, vb % 2)], self.lr))
            K.precondition_update_sliced(items)  # W -= eta B^-1 G A^-1, one grouped call
            done = torch.cuda.Event()
            done.record(self.compute)
            for l in range(ks.layers):
                for f in (0, 1):
                    v = ks.version[(l, f)]
                    if v >= 0:
                        ks.slot_free[(l, f, v % 2)] = done
        with torch.no_grad():
            for p in mod.parameters():
                if p.grad is not None and id(p) not in kfac_params:
                    p.add_(p.grad, alpha=-self.lr)
                p.grad = None
        self._end("PREC", e0, self.compute, stage=stage, step=step)

    def end_cycle(self):
        for mod in self.stages.values():
            mod.store.clear()


# ------------------------------------------------------------ measured costs
@dataclass
class MeasuredTimes:
    """Per-item device times (ms, CUDA events on the launching stream) of one
    hosted stage, the inputs of the assigner's CostTable."""
    f: float             # forward of one micro-batch (tape capture on)
    b: float             # backward of one micro-batch
    curv: float          # one curvature item: one layer's A- or B-set SYRKs, one micro-batch (max of the two)
    inv: float           # one inversion item: one layer's A- or B-set damped inverses (max of the two)
    prec: float          # precondition + update of the whole stage
    layers: int          # encoder layers per stage (l)
    stages_per_device: int
    param_bytes: int     # fp32 parameters of the stage (SyncGrad volume)
    factor_bytes: int    # fp32 factors of the stage (SyncCurvature volume)


def costs_from_times(t: MeasuredTimes, comm_alpha_ms: float = 0.01,
                     comm_bytes_per_ms: float = 3.0e8) -> S.CostTable:
    """Reference cost-table semantics: t_curv is
    charged per (layer, set, micro) item; an inversion item lasts t_inv / l,
    so t_inv = l x one set's inversion; t_prec is the per-DEVICE tail, split
    t_prec / spd per hosted stage.  Collective costs: alpha-beta model with
    the given NVLink estimates (bubblefill model_collective)."""
    return S.CostTable(t_f=t.f, t_b=t.b, t_curv=t.curv, t_inv=t.layers * t.inv,
                       t_prec=t.stages_per_device * t.prec, m_theta=t.param_bytes,
                       m_curv=t.factor_bytes, comm_alpha=comm_alpha_ms, comm_beta=comm_bytes_per_ms)


def project_pipeline(t: MeasuredTimes, cfg: S.PipelineConfig) -> dict:
    """Simulate `cfg` with the reference assigner from per-LAYER item costs
    measured on this GPU (one stage of t.layers layers): F/B and precondition
    scale with the layers per stage, curvature / inversion items are per layer
    already.  Returns the plain pipeline period (F/B only), the PipeFisher
    period (refresh cycle / refresh steps, K-FAC items in bubbles + tail), the
    refresh period and the simulated utilisation.  A projection, not a
    measurement."""
    spd = 2 if cfg.method == S.Method.Chimera else 1
    l = cfg.layers_per_stage
    per = lambda v: v / t.layers * l  # noqa: E731
    costs = costs_from_times(MeasuredTimes(f=per(t.f), b=per(t.b), curv=t.curv, inv=t.inv, prec=per(t.prec),
                                           layers=l, stages_per_device=spd,
                                           param_bytes=int(per(t.param_bytes)),
                                           factor_bytes=int(per(t.factor_bytes))))
    base = S.build_schedule(cfg, costs)
    plain_ms = S.schedule_metrics(base)[0]
    try:
        filled = S.assign_works(base, cfg, costs, S.enumerate_kfac_works(cfg, costs), S.AssignOptions())
    except S.InfeasibleError as e:
        return {"plain_step_ms": plain_ms, "infeasible": str(e)[:200]}
    span, util, _ = S.schedule_metrics(filled.schedule)
    period = span / filled.refresh_period
    return {"plain_step_ms": plain_ms, "pipefisher_step_ms": period, "step_ratio_vs_plain": period / plain_ms,
            "refresh_period": filled.refresh_period, "simulated_util": util,
            "cost_table": {k: getattr(costs, k) for k in ("t_f", "t_b", "t_curv", "t_inv", "t_prec")}}


def measure_stage_times(backend: "CudaBackend", reps: int = 3) -> MeasuredTimes:
    """Time the work items of this rank's first hosted stage.  Mutates the
    backend's model and K-FAC state: use a throw-away backend."""
    stage = min(backend.stages)
    backend.recompute_on = False  # t_f and t_b as such; the schedule adds t_f per Recompute item
    mod, ks = backend.stages[stage], backend.kstate[stage]
    topo = backend.topo
    micro = next(m for m in range(topo.cfg.micro_batches)
                 if topo.device(topo.pipe_of(m), stage, backend.rank // topo.D) == backend.rank)

    def timed(fn, stream):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        return e0, e1

    def median_ms(pairs):
        torch.cuda.synchronize(backend.device)
        v = sorted(a.elapsed_time(b) for a, b in pairs)
        return v[len(v) // 2]

    x = None if mod.is_first else torch.randn((backend.B, backend.Sq, backend.bert.hidden), device=backend.device,
                                              dtype=torch.bfloat16)
    gy = None if mod.is_last else torch.randn((backend.B, backend.Sq, backend.bert.hidden), device=backend.device,
                                              dtype=torch.bfloat16)
    fwd, bwd = [], []
    for i in range(reps + 1):  # first round warms cuBLAS / allocator
        pf = timed(lambda: backend.forward(stage, micro, None if x is None else x.clone(), True, 0), backend.compute)
        pb = timed(lambda: backend.backward(stage, micro, gy, True), backend.compute)
        if i:
            fwd.append(pf)
            bwd.append(pb)
        for p in mod.parameters():
            p.grad = None
    curv, inv = [], []
    for i in range(reps + 1):  # curvature first: no graph capture (synchronize, empty_cache) in between
        for f in (0, 1):
            pc = timed(lambda: backend.curvature_many([(stage, 0, f, micro)], None), backend.kfac_stream)
            if i:
                curv.append(pc)
    for i in range(reps + 2):  # round 0 captures the inversion graphs (graph_fb), round 1 uploads them
        for f in (0, 1):
            pi = timed(lambda: backend.invert_many([(stage, 0, f)], None), backend.kfac_stream)
            if i >= 2:
                inv.append(pi)
    t_curv = median_ms(curv[0::2]), median_ms(curv[1::2])
    t_inv = median_ms(inv[0::2]), median_ms(inv[1::2])
    if os.environ.get("PF_DEBUG_TIMES"):
        print("measure_stage_times inv", [a.elapsed_time(b) for a, b in inv],
              "curv", [a.elapsed_time(b) for a, b in curv], flush=True)
    prec = []
    for i in range(reps + 1):
        backend.forward(stage, micro, None if x is None else x.clone(), False, 0)
        backend.backward(stage, micro, gy, False)
        pp = timed(lambda: backend.precondition(stage, 0), backend.compute)
        if i:
            prec.append(pp)
    backend.end_cycle()
    backend.losses.clear()
    params = sum(p.numel() for p in mod.parameters()) * 4
    factors = sum(t.numel() for t in ks.factor.values()) * 4
    return MeasuredTimes(f=median_ms(fwd), b=median_ms(bwd), curv=max(t_curv), inv=max(t_inv),
                         prec=median_ms(prec), layers=topo.cfg.layers_per_stage,
                         stages_per_device=len(backend.stages), param_bytes=params, factor_bytes=factors)


@dataclass
class CycleResult:
    cycle_ms: float
    step_ms: float
    util: float
    busy_ms: float
    loss: Optional[float]


class PipeFisherTrainer:
    """Topology + schedule + program + backend for THIS rank."""

    def __init__(self, cfg: S.PipelineConfig, bert: BertConfig, rank: int = 0, world: int = 1,
                 device=None, kfac: bool = True, refresh: int = 2, costs: Optional[S.CostTable] = None,
                 damping: float = 0.1, lr: float = 1e-3, seed: int = 0, dist=None,
                 inversion_parallel: bool = False, graph_fb: bool = False):
        self.cfg, self.bert, self.rank, self.world = cfg, bert, rank, world
        self.topo = R.Topology(cfg)
        if self.topo.n_devices() != world:
            raise ValueError(f"config needs {self.topo.n_devices()} devices, world is {world}")
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.measured: Optional[MeasuredTimes] = None
        self._graph_fb = graph_fb
        if isinstance(costs, str):
            if costs != "measured":
                raise ValueError("costs: a CostTable or 'measured'")
            costs = self._measure_costs(damping, lr, seed, dist)
        self.costs = costs
        self.backend = CudaBackend(self.topo, bert, rank, self.device, kfac, damping, lr, seed, dist,
                                   graph_fb=graph_fb)
        self.filled = None
        if cfg.stages == 1 and cfg.replicas == 1:
            prog = R.inline_program(cfg, refresh)
            progs = [prog]
        else:
            costs = costs or S.CostTable(t_f=1.0, t_b=2.0, t_curv=0.05, t_inv=0.3, t_prec=0.1)
            base = S.build_schedule(cfg, costs)
            self.filled = S.assign_works(base, cfg, costs, S.enumerate_kfac_works(cfg, costs),
                                         S.AssignOptions(inversion_parallel=inversion_parallel))
            progs = R.device_programs(self.filled, cfg)  # inverse broadcast whenever W > 1
        if not kfac:
            progs = [[o for o in p if o.kind in (R.F_, R.RECOMP, R.B_, R.SYNC_GRAD, R.PREC)] for p in progs]
            for p in progs:
                R._assign_gates(p)
        self.programs = progs
        self.program = progs[rank]
        self.refresh = max((o.step for o in self.program), default=0) + 1
        self.comm = None
        if world > 1:
            replica_sets = [self.topo.replicas(s) for s in range(cfg.stages)]
            self.comm = R.Comm(dist, rank, R.channel_plan(progs), replica_sets, self.device)
        self.executor = R.Executor(self.program, self.backend, self.comm or _LocalComm(), rank)
        self.cycles = 0

    def _measure_costs(self, damping, lr, seed, dist) -> S.CostTable:
        """Profiler -> CostTable closed loop (the paper's 'collect the profile,
        then pick one work from the queue'): time the work
        items on a throw-away backend, take the max over ranks (every rank
        must build the identical schedule), convert to the reference's
        cost-table semantics."""
        probe = CudaBackend(self.topo, self.bert, self.rank, self.device, True, damping, lr, seed, dist,
                            graph_fb=self._graph_fb)
        t = measure_stage_times(probe)
        del probe
        torch.cuda.empty_cache()
        if dist is not None and self.world > 1:
            v = torch.tensor([t.f, t.b, t.curv, t.inv, t.prec, float(t.stages_per_device),
                              float(t.param_bytes), float(t.factor_bytes)], device=self.device, dtype=torch.float64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            t = MeasuredTimes(*[float(a) for a in v[:5].tolist()], layers=t.layers,
                              stages_per_device=int(v[5]), param_bytes=int(v[6]), factor_bytes=int(v[7]))
        self.measured = t
        torch.cuda.set_stream(torch.cuda.default_stream(self.device))
        return costs_from_times(t)

    def run_cycle(self, record: bool = False) -> CycleResult:
        b = self.backend
        b.record = record
        b.timeline.clear()
        b.losses.clear()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(b.compute)
        self.executor.run_cycle(self.cycles)
        if self.comm:
            self.comm.flush()
        b.compute.wait_stream(b.kfac_stream)
        t1.record(b.compute)
        torch.cuda.synchronize(self.device)
        self.cycles += 1
        cycle_ms = t0.elapsed_time(t1)
        busy = 0.0
        if record and b.timeline:
            iv = sorted((t0.elapsed_time(e0), t0.elapsed_time(e1)) for _, e0, e1, _ in b.timeline)
            self.last_trace = [(k, t0.elapsed_time(e0), t0.elapsed_time(e1), m) for k, e0, e1, m in b.timeline]
            self.last_cycle_ms = cycle_ms
            cur_b, cur_e = iv[0]
            for s, e in iv[1:]:
                if s > cur_e:
                    busy += cur_e - cur_b
                    cur_b, cur_e = s, e
                else:
                    cur_e = max(cur_e, e)
            busy += cur_e - cur_b
        loss = float(torch.stack(b.losses).mean()) if b.losses else None
        return CycleResult(cycle_ms, cycle_ms / self.refresh, busy / cycle_ms if cycle_ms > 0 else 0.0,
                           busy, loss)


def kernel_activity(trainer: "PipeFisherTrainer") -> dict:
    """One cycle under CUPTI (torch.profiler, CUDA activity only): the paper's
    GPU utilisation -- the fraction of the cycle in which SOME kernel runs on
    this device (reference definition over item intervals,
    schedule.cpp:257-270) -- measured from kernel execution intervals instead
    of the CUDA-event brackets of the ops (which cannot see host gaps inside
    an op).  Also splits the kernel time into this library's K-FAC kernels
    (pf::) and everything else (F/B, collectives, copies), and reports the
    idle time.  Profiler numbers: for explanation, not for the bench value."""
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize(trainer.device)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        trainer.run_cycle()
        torch.cuda.synchronize(trainer.device)
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    if not ev:
        return {"error": "no CUDA activity recorded"}
    ev.sort(key=lambda e: e.time_range.start)
    t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:
        a, b = e.time_range.start, e.time_range.end
        if cur_s is None or a > cur_e:
            if cur_s is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    busy += cur_e - cur_s
    kfac = sum(e.time_range.elapsed_us() for e in ev if "pf::" in e.name)
    other = sum(e.time_range.elapsed_us() for e in ev if "pf::" not in e.name)
    span = t1 - t0
    steps = max(1, trainer.refresh)
    return {"kernel_util": busy / span if span > 0 else 0.0, "span_ms": span / 1e3,
            "idle_ms_per_step": (span - busy) / 1e3 / steps,
            "kfac_kernel_ms_per_step": kfac / 1e3 / steps, "other_kernel_ms_per_step": other / 1e3 / steps,
            "kernels": len(ev),
            "definition": "union of CUDA kernel/memcpy execution intervals (CUPTI) / span of the cycle"}


_TRACE_KIND = {"F": S.WorkKind.Forward, "B": S.WorkKind.Backward, "RECOMP": S.WorkKind.Recompute,
               "CURV": S.WorkKind.Curvature,
               "INV": S.WorkKind.Inversion, "PREC": S.WorkKind.Precondition, "SYNC_GRAD": S.WorkKind.SyncGrad,
               "SYNC_CURV": S.WorkKind.SyncCurvature}


def _trace_event(kind, start_ms, dur_ms, device, devices_per_group, stage, step, micro=None, layer=None,
                 factor=None, extra=None):
    """One event of the reference trace schema (proj/src/io/trace.cpp:38-63):
    Chrome 'X' events, ts/dur in us, pid = replica group, tid = device, name
    'kind [lL] [A|B] [mM]' or 'kind sS'."""
    name = S.kind_name(kind)
    if layer is not None:
        name += f" l{layer}"
    if factor is not None:
        name += " " + ("A" if int(factor) == 0 else "B")
    if micro is not None:
        name += f" m{micro}"
    if layer is None and factor is None and micro is None:
        name += f" s{stage}"
    args = {"kind": S.kind_name(kind), "stage": stage, "step": step}
    if micro is not None:
        args["micro_batch"] = micro
    if layer is not None:
        args["layer"] = layer
    if factor is not None:
        args["factor"] = "A" if int(factor) == 0 else "B"
    if extra:
        args.update(extra)
    def llround(v):  # std::llround: halves away from zero
        return int(math.floor(abs(v) + 0.5)) * (1 if v >= 0 else -1)

    return {"name": name, "ph": "X", "ts": llround(start_ms * 1000.0), "dur": llround(dur_ms * 1000.0),
            "pid": device // devices_per_group if devices_per_group > 0 else 0, "tid": device, "args": args}


def schedule_trace(schedule: S.StaticSchedule, devices_per_group: int = 0) -> dict:
    """The reference's trace_to_json for a (simulated) schedule."""
    ev = []
    for d, line in enumerate(schedule.timelines):
        for it in line:
            ev.append(_trace_event(it.kind, it.start, it.duration, d, devices_per_group, it.stage, it.step,
                                   it.micro_batch, it.layer, it.factor))
    return {"traceEvents": ev}


def measured_trace(trainer: "PipeFisherTrainer") -> dict:
    """The last recorded cycle (run_cycle(record=True)) of this rank as MEASURED
    intervals (CUDA events on the launching streams) in the same schema, plus
    utilisation by the reference definition (schedule.cpp:257-270: sum of item
    durations / (makespan x devices)) and by the union of busy intervals (the
    K-FAC stream overlaps the compute stream, so the sum can exceed the span)."""
    ev, busy_sum = [], 0.0
    for kind, a, b, m in getattr(trainer, "last_trace", []):
        extra = {"items": m["items"]} if "items" in m else None
        ev.append(_trace_event(_TRACE_KIND[kind], a, b - a, trainer.rank, trainer.topo.D, m.get("stage", -1),
                               m.get("step", 0), m.get("micro_batch"), m.get("layer"), m.get("factor"), extra))
        busy_sum += b - a
    span = getattr(trainer, "last_cycle_ms", 0.0)
    return {"traceEvents": ev,
            "otherData": {"source": "measured: CUDA events around each op on its stream (batched items = one event)",
                          "cycle_ms": span, "refresh_steps": trainer.refresh,
                          "util_reference_definition": busy_sum / span if span > 0 else 0.0}}


def _overlap(a, b, iv):
    """Length of [a, b] covered by the sorted, disjoint intervals iv."""
    return sum(max(0.0, min(b, e) - max(a, s)) for s, e in iv if e > a and s < b)


def _union(iv):
    out = []
    for s, e in sorted(iv):
        if out and s <= out[-1][1]:
            out[-1][1] = max(out[-1][1], e)
        else:
            out.append([s, e])
    return [(s, e) for s, e in out]


def bubble_landing(program, trace, cycle_ms: float) -> dict:
    """Where the K-FAC items of one recorded cycle actually ran against the
    bubbles the assigner gave them (bubblefill.cpp:286-344 places each item in
    a gap of its device's timeline; runtime._assign_gates turns that gap into
    'after F/B op g, before the next F/B op').

    program: the device program (runtime.Op list, schedule-time costs);
    trace: [(kind, start_ms, end_ms, meta)] of run_cycle(record=True), meta
    carrying the program index ('op') and gate ('gate') of each event.

    Per bubble (the gate op): its planned length (schedule units), its
    measured length (end of the gate F/B -> start of the next F/B on the
    compute stream, or the cycle end), the K-FAC time that ran inside it and
    the part that spilled past it (running beside the next F/B).  Totals: the
    fraction of K-FAC time inside its own bubble, the fraction that overlapped
    ANY F/B, and the count of items that started before their gate ended (a
    dependency violation; must be 0)."""
    fb = {}
    for kind, a, b, m in trace:
        if kind in COMPUTE_KINDS and m.get("op") is not None:
            s, e = fb.get(m["op"], (a, b))
            fb[m["op"]] = (min(s, a), max(e, b))
    fb_iv = _union(fb.values())
    compute_idx = [i for i, o in enumerate(program) if o.kind in COMPUTE_KINDS]
    bubbles: Dict[object, dict] = {}
    eps = 1e-3  # ms: event timestamp resolution
    early = 0
    for kind, a, b, m in trace:
        if kind not in KFAC_KINDS:
            continue
        g = m.get("gate")
        b0 = fb[g][1] if g is not None and g in fb else 0.0
        nxt = next((i for i in compute_idx if g is None or i > g), None)
        b1 = fb[nxt][0] if nxt is not None and nxt in fb else cycle_ms
        if g is not None and nxt is not None:
            go, no = program[g], program[nxt]
            planned = no.start - (go.start + go.duration)
        elif nxt is not None:
            planned = program[nxt].start
        else:
            planned = None
        if a < b0 - eps:
            early += 1
        bub = bubbles.setdefault(g, {"gate": g, "next": nxt, "planned": planned, "measured_ms": max(0.0, b1 - b0),
                                     "begin": b0, "end": b1, "items": 0, "iv": [], "kinds": []})
        bub["items"] += int(m.get("items", 1))
        bub["iv"].append((a, b))
        bub["kinds"].append(kind)
    rows, k_total, k_inside, k_fb = [], 0.0, 0.0, 0.0
    for g in sorted(bubbles, key=lambda x: -1 if x is None else x):
        bub = bubbles[g]
        iv = _union(bub.pop("iv"))
        busy = sum(e - s for s, e in iv)
        inside = sum(_overlap(bub["begin"], bub["end"], [(s, e)]) for s, e in iv)
        with_fb = sum(_overlap(s, e, fb_iv) for s, e in iv)
        k_total, k_inside, k_fb = k_total + busy, k_inside + inside, k_fb + with_fb
        bub.update(kfac_ms=busy, inside_ms=inside, spill_ms=busy - inside, kinds=sorted(set(bub["kinds"])))
        rows.append(bub)
    return {"bubbles": rows, "kfac_ms": k_total,
            "inside_fraction": k_inside / k_total if k_total > 0 else 1.0,
            "fb_overlap_fraction": k_fb / k_total if k_total > 0 else 0.0,
            "started_before_gate": early}


def trainer_bubble_landing(trainer: "PipeFisherTrainer") -> dict:
    """bubble_landing of this rank's last run_cycle(record=True)."""
    return bubble_landing(trainer.program, getattr(trainer, "last_trace", []),
                          getattr(trainer, "last_cycle_ms", 0.0))


COMPUTE_KINDS = ("F", "RECOMP", "B")
KFAC_KINDS = ("CURV", "SYNC_CURV", "INV")


class _LocalComm:
    def group(self, devs):
        return None

    def flush(self):
        pass
