#!/usr/bin/env python
"""PipeFisher B200 benchmark (contract: one JSON line on rank 0).

Workload (config.workload = "bert_large_kfac_layer_step"): one K-FAC step of
one BERT-Large encoder layer — BASELINE.json configs[0] at BERT-Large shapes
(hidden 1024, FFN 4096, micro-batch 32 x 128 = 4096 tokens), the per-layer
unit of the Chimera/1F1B configs the metric is quoted on:
  * curvature: 12 Kronecker factors (A and B of Q, K, V, O, FFN1, FFN2;
    10 x 1024^2 + 2 x 4096^2) from bf16 tapes, one grouped tcgen05 SYRK launch;
  * inversion: 12 damped inverses (lambda = 0.1), fp32-accurate, batched;
  * precondition: 6 x  W -= eta B^-1 G A^-1  (fp32-accurate int8-digit tcgen05 GEMMs, fused update).
Algorithmic FLOPs per step: SYRK d(d+1)n, inverse d^3,
precondition 2 d_out^2 d_in + 2 d_out d_in^2.  value = those FLOPs / step time.

N > 1 (torchrun, one rank per GPU): data-parallel replicas of the layer step
with the path's real exchange steps — factor all-reduce (SyncCurvature) over
NCCL and inversion parallelism (round-robin inversion ownership, inverse
broadcast) as in the paper; weak scaling.

--impl reference: the reference's own CPU implementation (oracle/_ref, the
unmodified reference sources compiled in-tree) on the same metric, a bounded
sample per step, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BERT-Large PipeFisher step time & GPU util at 1/2/4/8 B200; K-FAC TFLOP/s"
UNIT = "TFLOP/s"
D_MODEL, D_FF, TOKENS = 1024, 4096, 32 * 128
LINEARS = [("q", D_MODEL, D_MODEL), ("k", D_MODEL, D_MODEL), ("v", D_MODEL, D_MODEL),
           ("o", D_MODEL, D_MODEL), ("ffn1", D_MODEL, D_FF), ("ffn2", D_FF, D_MODEL)]  # (name, d_in, d_out)
DAMPING, ETA = 0.1, 1e-3


def layer_flops(tokens=TOKENS):
    syrk = sum(d * (d + 1) * tokens for _, di, do in LINEARS for d in (di, do))
    inv = sum(d ** 3 for _, di, do in LINEARS for d in (di, do))
    prec = sum(2 * do * do * di + 2 * do * di * di for _, di, do in LINEARS)
    return syrk, inv, prec


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                f = [x.strip() for x in out.split(",")]
                if len(f) >= 7:
                    self.samples.append(f)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if s[3 + i].lower() in ("active", "1", "yes")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ====================================================================== CPU arms
def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def reference_sample(threads):
    """A bounded sample of the same layer step on the reference CPU path
    (oracle/_ref = the unmodified reference sources): per thread one item of
    each kind at BERT-Large d_model size with the FULL micro-batch -- one
    curvature factor over all 4096 tokens (kfac.cpp:125-131), one
    cholesky_spd_inverse(1024) (matrix.cpp:136-163) and one
    precondition(1024 x 1024) (kfac.cpp:133-137) -- timed once on one core and
    then on `threads` cores at once (independent calls, std::thread-parallel
    through the GIL-free ctypes calls).  The layer's two d = 4096 inverses are
    NOT in the sample: one takes ~426 s single-threaded (BASELINE.md §2, 0.16
    GF/s against 0.30 GF/s at d = 1024), so the sampled rate flatters the CPU.
    Returns (rate on `threads` cores, seconds, 1-core rate, sample text)."""
    from oracle import ref as R
    a = R.orc_symmetric(1, (D_MODEL, TOKENS), 3 ** 0.5)
    e = R.orc_symmetric(2, (1, TOKENS), 3 ** 0.5)  # B of a 1-wide layer: negligible
    g = R.orc_symmetric(3, (D_MODEL, D_MODEL))

    def job(_):
        t0 = time.perf_counter()
        F, _ = R.ref_curvature_factors(a, e)
        ai = R.ref_cholesky_spd_inverse(F, DAMPING)
        R.ref_precondition(g, ai, ai)
        return time.perf_counter() - t0

    flops_per_job = D_MODEL * (D_MODEL + 1) * TOKENS + D_MODEL ** 3 + 4 * D_MODEL ** 3
    one = job(0)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(job, range(threads)))
    dt = time.perf_counter() - t0
    sample = (f"per core: curvature_factors({D_MODEL} x {TOKENS} tokens) + cholesky_spd_inverse({D_MODEL})"
              f" + precondition({D_MODEL}x{D_MODEL}), FP64; {threads} cores = independent calls "
              f"(std::thread via ctypes); 1 core timed alone first; the layer's 4096-wide factors are not "
              f"sampled (one d=4096 inverse: ~426 s on one core) -- the sampled rate flatters the CPU")
    return threads * flops_per_job / dt / 1e12, dt, flops_per_job / one / 1e12, sample


def int8_peaks():
    """Measured dense int8 peak on this GPU model (tools/int8_peak.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "int8_peak.json")) as f:
            return json.load(f)
    except Exception:
        return {"int8_tops_burst": 3089.3, "int8_tops_sustained": 2407.6}


def cpu_threads():
    try:
        return max(1, min(len(os.sched_getaffinity(0)), 16))
    except Exception:
        return max(1, min(os.cpu_count() or 1, 16))


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    threads = cpu_threads()
    for _ in range(args.warmup):
        reference_sample(threads)
    vals, times, ones = [], [], []
    for _ in range(args.steps):
        v, dt, v1, sample = reference_sample(threads)
        vals.append(v)
        times.append(dt)
        ones.append(v1)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SplitMix64)",
        "config": {"workload": "bert_large_kfac_layer_step", "sample": "bounded CPU sample",
                   "tokens": TOKENS, "d": D_MODEL},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample, "value_1core": statistics.mean(ones), "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ====================================================================== GPU arm
class LayerStep:
    """Device-resident state for one replica's layer step."""

    def __init__(self, torch, K, seed):
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.torch, self.K = torch, K
        self.tapes, self.factors, self.inv, self.digits = [], [], [], []
        for _, di, do in LINEARS:
            for d in (di, do):
                # token-major [tokens x d]: a layer's activations / output
                # gradients as produced, read in place by the SYRK (MN-major)
                self.tapes.append(torch.randn((TOKENS, d), generator=g, device="cuda").to(torch.bfloat16))
                self.factors.append(torch.empty((d, d), device="cuda"))
                self.inv.append(torch.empty((d, d), device="cuda"))
                self.digits.append(torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda"))
        self.grads = [torch.randn((do, di), generator=g, device="cuda") for _, di, do in LINEARS]
        self.weights = [0.02 * torch.randn((do, di), generator=g, device="cuda") for _, di, do in LINEARS]

    def curvature(self):
        self.K.syrk([(x, f, 1.0 / TOKENS, False, True) for x, f in zip(self.tapes, self.factors)],
                    fill_upper=False)

    def invert(self, which=None):
        idx = range(len(self.factors)) if which is None else which
        idx = list(idx)
        if idx:
            self.K.damped_inverse_batched([self.factors[i] for i in idx], DAMPING,
                                          [self.inv[i] for i in idx],
                                          [self.digits[i] for i in idx], check=False)

    def precondition(self):
        K = self.K
        items = []
        for l in range(len(LINEARS)):
            ai = K.SlicedMatrix(self.inv[2 * l], self.digits[2 * l])
            bi = K.SlicedMatrix(self.inv[2 * l + 1], self.digits[2 * l + 1])
            items.append((self.weights[l], self.grads[l], ai, bi, ETA))
        K.precondition_update_sliced(items)


def sync_factors(torch, dist, factors, tril):
    """SyncCurvature of the N > 1 layer step: the replica average of the
    factors.  The SYRK writes lower tiles only, so the packed lower triangles
    of all factors travel in ONE all-reduce (sum d(d+1)/2 floats: 88 MB for the
    BERT-Large layer instead of 168 MB of full squares in 12 calls)."""
    packed = torch.cat([f.view(-1).index_select(0, i) for f, i in zip(factors, tril)])
    dist.all_reduce(packed, op=dist.ReduceOp.AVG)
    off = 0
    for f, i in zip(factors, tril):
        f.view(-1).index_copy_(0, i, packed[off:off + i.numel()])
        off += i.numel()


def share_inverses(dist, digits, world):
    """Inversion parallelism: factor i was inverted on rank i % world; only its
    digit form travels (all the preconditioner reads), as asynchronous
    broadcasts waited together."""
    works = [dist.broadcast(dg, src=i % world, async_op=True) for i, dg in enumerate(digits)]
    for w in works:
        w.wait()


def self_check(torch, st, step_a, step_b, owned=None):
    """The bench checks its OWN step (outside the timed region), in fp64 on the
    device: the damped-inverse residual max|(A + lambda I) X - I| of every
    factor the step inverted (reference norm, proj/tests/test_kfac.cpp:155;
    north_star bound 1e-5), and the fused update W -= eta B^-1 G A^-1 of every
    linear against the same update formed with fp64 inverses of the step's
    own factors (relative Frobenius; north_star bound 1e-3)."""
    step_a()
    torch.cuda.synchronize()
    f64 = torch.float64
    damped, resid = [], {}
    for i, (f, x) in enumerate(zip(st.factors, st.inv)):
        d = f.shape[0]
        a = f.to(f64)
        a = torch.tril(a) + torch.tril(a, -1).T + DAMPING * torch.eye(d, device=f.device, dtype=f64)
        damped.append(a)
        if owned is not None and i not in owned:
            continue  # inverted on another rank (only its digit form travels)
        r = (a @ x.to(f64) - torch.eye(d, device=f.device, dtype=f64)).abs().max().item()
        resid[str(d)] = max(resid.get(str(d), 0.0), r)
    w0 = [w.clone() for w in st.weights]
    step_b()
    torch.cuda.synchronize()
    rel = 0.0
    for l in range(len(LINEARS)):
        ai = torch.linalg.inv(damped[2 * l])
        bi = torch.linalg.inv(damped[2 * l + 1])
        want = -ETA * (bi @ st.grads[l].to(f64) @ ai)
        got = st.weights[l].to(f64) - w0[l].to(f64)
        rel = max(rel, ((got - want).norm() / want.norm()).item())
    return {"inverse_residual_max": resid, "inverse_residual_bound": 1e-5,
            "update_rel_fro_max": rel, "update_rel_fro_bound": 1e-3,
            "ok": max(resid.values(), default=0.0) <= 1e-5 and rel <= 1e-3,
            "how": "fp64 on the device, after the timed region, on the step's own factors / inverses / weights"}


def run_gpu_arm(args, rank, world, local_rank):
    import torch
    from paper_2211_14133_b200 import kfac as K
    torch.cuda.set_device(local_rank)
    if not K.device_ok():
        raise SystemExit("libpf_b200.so: no sm_100 device")
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))

    st = LayerStep(torch, K, seed=1234 + rank)
    stream = torch.cuda.current_stream()

    tril = None
    if world > 1:
        from paper_2211_14133_b200.engine import _tril_index
        tril = [_tril_index(f.shape[0], f.device) for f in st.factors]

    def exchange():
        sync_factors(torch, dist, st.factors, tril)

    def step(ev=None):
        step_a(ev)
        step_b(ev)

    def step_a(ev=None):  # needs the tapes
        if ev: ev[0].record(stream)
        st.curvature()
        if ev: ev[1].record(stream)
        if world > 1:
            exchange()
            # inversion parallelism: factor i inverted on rank i % world; only
            # the digit form travels (all the preconditioner reads), as
            # asynchronous broadcasts waited together
            mine = [i for i in range(len(st.factors)) if i % world == rank]
            st.invert(mine)
            share_inverses(dist, st.digits, world)
        else:
            st.invert()
        if ev: ev[2].record(stream)

    def step_b(ev=None):  # needs the gradients
        st.precondition()
        if ev: ev[3].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    # One layer step = ~400 small launches (the inversion recursion): the
    # single-GPU step is captured once as a CUDA graph and replayed, so host
    # enqueue cost never shows up as GPU idle time.  (N > 1 interleaves NCCL
    # calls and runs eagerly.)
    run = step
    graphed = False
    if world == 1 and not args.no_graph:
        launches_per_step = K.kernel_launches()
        step()
        torch.cuda.synchronize()
        launches_per_step = K.kernel_launches() - launches_per_step
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        graph.replay()
        torch.cuda.synchronize()
        run = graph.replay
        graphed = True

    # ---------------------------------------------------------- device timing
    if dist: dist.barrier()
    torch.cuda.synchronize()
    launches0 = K.kernel_launches()
    with ClockSampler(local_rank) as clocks:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            run()
        t_end.record(stream)
        torch.cuda.synchronize()
    launches = K.kernel_launches() - launches0
    if graphed:
        launches = launches_per_step * args.steps  # replays do not pass through the host counter
    if dist: dist.barrier()
    ms = t_start.elapsed_time(t_end) / args.steps

    # phase breakdown.  Graphed: replays of the step's prefixes (curvature;
    # curvature + inversion; the whole step), each timed alone with events, so
    # the phases are measured as the step runs (the inversion's ~300 launches
    # are host-bound when issued eagerly).  Otherwise an eager pass with events
    # between the phases.
    phases = {"curvature": 0.0, "inversion": 0.0, "precondition": 0.0}
    if graphed:
        def prefix_graph(fn):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                fn()
            return g

        g_c = prefix_graph(st.curvature)
        g_ci = prefix_graph(lambda: (st.curvature(), st.invert()))

        def replay_ms(g):
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / args.steps

        t_c, t_ci, t_all = replay_ms(g_c), replay_ms(g_ci), replay_ms(graph)
        phases = {"curvature": t_c, "inversion": t_ci - t_c, "precondition": t_all - t_ci}
    else:
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        for i in range(args.steps):
            step(evs[i])
        torch.cuda.synchronize()
        for e in evs:
            phases["curvature"] += e[0].elapsed_time(e[1]) / args.steps
            phases["inversion"] += e[1].elapsed_time(e[2]) / args.steps
            phases["precondition"] += e[2].elapsed_time(e[3]) / args.steps
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    syrk_f, inv_f, prec_f = layer_flops()
    job_flops = world * (syrk_f + prec_f) + inv_f * (1 if world > 1 else 1)
    if world == 1:
        job_flops = syrk_f + inv_f + prec_f
    value = job_flops / (ms * 1e-3) / 1e12

    # ---------------------------------------------------------- end-to-end (public API, host buffers)
    # Every step copies its tapes + gradients from pinned host memory and reads
    # the updated weights back; the copies of neighbouring steps overlap the
    # compute (double-buffered device inputs, copy engines on their own
    # streams): H2D(k+1) || compute(k) || D2H(k-1).  All of it is inside the
    # timed region.
    # Inputs and outputs are packed into ONE pinned host buffer each way and
    # the device tensors are views of one buffer per double-buffer slot, so
    # every step is one H2D and one D2H copy (18 separate copies per step
    # cost ~0.4 ms of per-copy overhead on a copy engine that is already the
    # e2e bound: 201 MB at ~55 GB/s).
    def packed(tensors):
        offs, total = [], 0
        for t in tensors:
            offs.append(total)
            total += (t.numel() * t.element_size() + 255) // 256 * 256
        return offs, total

    def views(buf, tensors, offs):
        return [buf[o:o + t.numel() * t.element_size()].view(t.dtype).view(t.shape) for t, o in zip(tensors, offs)]

    ins = list(st.tapes) + list(st.grads)
    in_offs, in_total = packed(ins)
    h_in = torch.empty(in_total, dtype=torch.uint8).pin_memory()
    for hv, t in zip(views(h_in, ins, in_offs), ins):
        hv.copy_(t.cpu())
    out_offs, out_total = packed(st.weights)
    h_out = torch.empty(out_total, dtype=torch.uint8).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in ins)
    d2h = sum(t.numel() * t.element_size() for t in st.weights)
    d_in = [torch.empty(in_total, dtype=torch.uint8, device="cuda") for _ in (0, 1)]
    sets = []
    for buf in d_in:
        vs = views(buf, ins, in_offs)
        for v, t in zip(vs, ins):
            v.copy_(t)
        sets.append((vs[:len(st.tapes)], vs[len(st.tapes):]))
    d_out = [torch.empty(out_total, dtype=torch.uint8, device="cuda") for _ in (0, 1)]
    w_snaps = [views(buf, st.weights, out_offs) for buf in d_out]
    copy_in = torch.cuda.Stream()
    copy_out = torch.cuda.Stream()

    def use(k):
        st.tapes, st.grads = sets[k % 2]

    def snapshot(k):
        for w, sw in zip(st.weights, w_snaps[k % 2]):
            sw.copy_(w)

    # each step in two parts: curvature + inversion need only the tapes, the
    # preconditioner the gradients, so the first step starts once its tapes
    # (3/4 of the bytes) are in and the gradients' copy overlaps the inversion
    runners = []
    for k in (0, 1):
        use(k)
        if world == 1 and not args.no_graph:
            ga, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
            with torch.cuda.graph(ga):
                step_a()
            with torch.cuda.graph(gb):
                step_b()
                snapshot(k)
            runners.append((ga.replay, gb.replay))
        else:
            runners.append((step_a, lambda k=k: (step_b(), snapshot(k))))
    torch.cuda.synchronize()
    n_tape_bytes = in_offs[len(st.tapes)] if len(st.grads) else in_total

    def h2d_into(k):
        evs = []
        with torch.cuda.stream(copy_in):
            d_in[k % 2][:n_tape_bytes].copy_(h_in[:n_tape_bytes], non_blocking=True)
            evs.append(torch.cuda.Event())
            evs[-1].record(copy_in)
            d_in[k % 2][n_tape_bytes:].copy_(h_in[n_tape_bytes:], non_blocking=True)
            evs.append(torch.cuda.Event())
            evs[-1].record(copy_in)
        return evs

    def e2e_run(n):
        in_ready = [h2d_into(0)]
        done, out_done = [], []
        for k in range(n):
            stream.wait_event(in_ready[k][0])
            if k >= 2:                     # weight snapshot buffer k%2 read back by step k-2's D2H
                stream.wait_event(out_done[k - 2])
            use(k)
            runners[k % 2][0]()
            stream.wait_event(in_ready[k][1])
            runners[k % 2][1]()
            ev = torch.cuda.Event()
            ev.record(stream)
            done.append(ev)
            if k + 1 < n:                  # next inputs: that buffer was last read by step k-1
                if k >= 1:
                    copy_in.wait_event(done[k - 1])
                in_ready.append(h2d_into(k + 1))
            copy_out.wait_event(ev)
            with torch.cuda.stream(copy_out):
                h_out.copy_(d_out[k % 2], non_blocking=True)
            od = torch.cuda.Event()
            od.record(copy_out)
            out_done.append(od)
        stream.wait_event(out_done[-1])

    e2e_run(2)
    if dist: dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if os.environ.get("PF_BENCH_E2E_TRACE") and rank == 0:  # development: copy/compute timeline
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            e2e_run(4)
            torch.cuda.synchronize()
        prof.export_chrome_trace(os.environ["PF_BENCH_E2E_TRACE"])
    use(0)
    if dist:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = job_flops / (e2e_ms * 1e-3) / 1e12

    check = self_check(torch, st, step_a, step_b,
                       owned=None if world == 1 else {i for i in range(len(st.factors)) if i % world == rank})
    if rank != 0:
        if not args.no_pipeline:
            with _Watchdog(world, None):
                pipeline_section(args, rank, world, local_rank, dist)
        if dist: dist.destroy_process_group()
        return

    pk, pk_kind = peaks()
    i8 = int8_peaks()
    prof = {}
    try:
        with open(os.path.join(ROOT, "profiles", "syrk_traffic.json")) as f:
            prof["syrk"] = json.load(f).get("dram_bytes_per_launch")
        with open(os.path.join(ROOT, "profiles", "digit_gemm_traffic.json")) as f:
            prof["digit"] = json.load(f).get("dram_bytes_per_launch")
        with open(os.path.join(ROOT, "profiles", "inversion_traffic.json")) as f:
            prof["inversion"] = json.load(f).get("dram_bytes_per_call")
    except Exception:
        pass
    # Every phase is timed ALONE (graph-prefix replays, a few ms each), so its
    # denominator is the BURST peak.  The fp32-accurate digit GEMM runs 10
    # int8 products per fp32 product: its ceiling is the measured dense int8
    # peak (cuBLASLt int8 8192^3, profiles/int8_peak.json) / 10.
    digit_peak = i8["int8_tops_burst"] / 10.0
    inv_ms, prec_ms, syrk_ms = phases["inversion"], phases["precondition"], phases["curvature"]
    inv_rate = inv_f / (inv_ms * 1e-3) / 1e12
    # The dominant phase (~80 % of the step) is the damped inversion: a chain
    # of leaf (SIMT 128x128 Cholesky + inverse), slicing and digit-GEMM
    # launches, so it is reported as a phase against the digit-GEMM ceiling.
    roof = {"kernel": "damped inversion phase (12 factors: 2 x 4096 + 10 x 1024; leaves + digit GEMMs + "
                      "slicing, one CUDA graph) -- the dominant phase",
            "bound": "tensor", "achieved": inv_rate, "peak": digit_peak, "unit": "TFLOP/s (fp32-equivalent)",
            "frac": inv_rate / digit_peak, "traffic": prof.get("inversion"),
            "traffic_note": "per call, all 516 kernels, ncu with caches flushed per kernel (profiles/inversion_traffic.json); algorithmic ~0.56 GB",
            "algorithmic": "d^3 per factor (POTRF d^3/3 + TRTRI d^3/3 + LAUUM d^3/3): 148.0 GFLOP",
            "share_of_step": inv_ms / ms if ms > 0 else None,
            "peak_source": "measured int8 dense burst (cuBLASLt, profiles/int8_peak.json) / 10 digit products"}
    syrk_rate = syrk_f / (syrk_ms * 1e-3) / 1e12
    roof_syrk = {"kernel": "umma_gemm_kernel<bf16> (grouped SYRK, 12 factors, 1 launch)",
                 "bound": "tensor", "achieved": syrk_rate, "peak": pk["bf16_tflops"],
                 "unit": "TFLOP/s", "frac": syrk_rate / pk["bf16_tflops"],
                 "traffic": prof.get("syrk"), "peak_source": f"{pk_kind} bf16_tflops (burst)"}
    int8_achieved = 10 * prec_f / (prec_ms * 1e-3) / 1e12
    roof_prec = {"kernel": "umma_gemm_persist_kernel (kOZ8 digit GEMM; precondition phase: 2 GEMM + 2 slice launches)",
                 "bound": "tensor", "achieved": int8_achieved, "peak": i8["int8_tops_burst"],
                 "unit": "TOP/s (int8)", "frac": int8_achieved / i8["int8_tops_burst"],
                 "traffic": prof.get("digit"),
                 "algorithmic": "10 int8 products x (2 d_out^2 d_in + 2 d_out d_in^2) per linear, 6 linears = 1.03 int8-POP",
                 "peak_source": "measured int8 dense burst (cuBLASLt 8192^3, profiles/int8_peak.json)"}
    phase_rates = {
        "curvature": {"ms": syrk_ms, "tflops": syrk_rate},
        "inversion": {"ms": inv_ms, "tflops": inv_rate, "peak_fp32_digit_tflops": digit_peak},
        "precondition": {"ms": prec_ms, "tflops": prec_f / prec_ms / 1e9, "peak_fp32_digit_tflops": digit_peak},
    }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        v, dt, v1, sample = reference_sample(threads)
        cpu = {"value": v, "unit": UNIT, "cores": threads, "kind": "reference", "sample": sample,
               "seconds": dt, "value_1core": v1, "cpu_model": cpu_model()}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16 curvature / fp32-accurate (int8-digit tcgen05) inversion+precondition",
        "data": "synthetic (torch.randn tapes/grads/weights, random init)",
        "config": {"workload": "bert_large_kfac_layer_step", "d_model": D_MODEL, "d_ff": D_FF,
                   "tokens_per_micro_batch": TOKENS, "factors": 12, "linears": 6,
                   "damping": DAMPING, "parallelism": f"dp{world}" + ("+inv-parallel" if world > 1 else ""),
                   "l2": "inputs larger than L2 (tapes 144 MB + factors 168 MB per step)"},
        "phases": phase_rates,
        "cuda_graph": graphed,
        "roofline": roof,
        "roofline_syrk": roof_syrk,
        "roofline_precondition": roof_prec,
        "check": check,
        "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "overlap": "pinned host buffers, one H2D for the tapes and one for the gradients per step (curvature + inversion start on the tapes, the preconditioner waits for the gradients), one D2H of the updated weights; H2D(step k+1) || compute(k) || D2H(k-1), double-buffered inputs; the copy engine (201 MB at ~55 GB/s) bounds the steady state"},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
        "pipeline": None,
    }
    if not args.no_pipeline:
        with _Watchdog(world, line):
            line["pipeline"] = pipeline_section(args, rank, world, local_rank, dist)
    print(json.dumps(line), flush=True)
    if dist: dist.destroy_process_group()


class _Watchdog:
    """N > 1: the pipeline section runs real NCCL point-to-point programs
    across ranks; if one rank fails inside them the others block in a
    collective for good.  After PF_BENCH_PIPE_TIMEOUT seconds (default 600)
    every rank exits, rank 0 first printing the bench line with the pipeline
    section marked as timed out -- a hang there never swallows the layer-step
    measurement.  N = 1 runs unguarded."""

    def __init__(self, world, line):
        self.world, self.line, self.timer = world, line, None

    def _fire(self):
        if self.line is not None:
            self.line["pipeline"] = {"error": "timed out (a rank failed or hung inside the pipeline programs)"}
            print(json.dumps(self.line), flush=True)
        os._exit(0)

    def __enter__(self):
        if self.world > 1:
            import threading
            self.timer = threading.Timer(float(os.environ.get("PF_BENCH_PIPE_TIMEOUT", "600")), self._fire)
            self.timer.daemon = True
            self.timer.start()
        return self

    def __exit__(self, *exc):
        if self.timer is not None:
            self.timer.cancel()
        return False


# ====================================================================== pipeline step
PIPELINE_LADDER = {  # SURVEY §8d 1/2/4/8-GPU ladder (BERT-Large, micro-batch 32 x 128)
    1: dict(method="gpipe", stages=1, micro_batches=4, replicas=1),      # inline K-FAC (no bubbles)
    2: dict(method="gpipe", stages=2, micro_batches=4, replicas=1),
    4: dict(method="gpipe", stages=4, micro_batches=4, replicas=1),
    8: dict(method="chimera", stages=8, micro_batches=8, replicas=2),    # BASELINE configs[2]
}


def pipeline_section(args, rank, world, local_rank, dist):
    import torch
    from paper_2211_14133_b200 import schedule as S
    from paper_2211_14133_b200.bert import BertConfig
    from paper_2211_14133_b200.engine import PipeFisherTrainer
    spec = PIPELINE_LADDER.get(world)
    if spec is None:
        return {"skipped": f"no ladder entry for {world} GPUs"}
    bert = BertConfig.large()
    method = S.parse_method(spec["method"])
    spd = 2 if method == S.Method.Chimera else 1
    L = bert.layers // spec["stages"]
    cfg = S.PipelineConfig(method=method, stages=spec["stages"], micro_batches=spec["micro_batches"],
                           micro_batch_size=32, replicas=spec["replicas"], layers_per_stage=L, seq_len=128)
    costs_box = {"costs": "measured"}  # profiler -> CostTable closed loop (engine.measure_stage_times)
    t_meas = {}
    out = {"model": "BERT-Large (24 x 1024, FFN 4096, 16 heads), random init", "method": spec["method"],
           "stages": cfg.stages, "micro_batches": cfg.micro_batches, "micro_batch": "32 x 128",
           "replicas": cfg.replicas, "layers_per_stage": L, "data": "synthetic token ids, 15% MLM"}

    def measure(kfac):
        t = PipeFisherTrainer(cfg, bert, rank, world, torch.device("cuda", local_rank), kfac=kfac,
                              refresh=2, costs=costs_box["costs"], dist=dist, seed=11, graph_fb=True)
        if t.measured is not None:
            m = t.measured
            t_meas["times"] = m
            costs_box["costs"] = t.costs
            costs_box["measured"] = {"t_f_ms": m.f, "t_b_ms": m.b, "curvature_item_ms": m.curv,
                                     "inversion_item_ms": m.inv, "precondition_stage_ms": m.prec,
                                     "cost_table": {k: getattr(t.costs, k) for k in
                                                    ("t_f", "t_b", "t_curv", "t_inv", "t_prec")},
                                     "source": "CUDA events on this GPU, median of 3, max over ranks"}
        for _ in range(2):  # warm-up (allocations, cuBLAS heuristics, F/B and inversion graph captures)
            t.run_cycle()
        if dist: dist.barrier()
        res = [t.run_cycle(record=(i == 1)) for i in range(2)]
        step = statistics.mean(r.step_ms for r in res)
        util = res[1].util
        info = {"refresh_period": t.refresh}
        try:  # the paper's utilisation from kernel activity (CUPTI), beside the event-bracket one
            from paper_2211_14133_b200.engine import kernel_activity
            info["cupti"] = kernel_activity(t)
        except Exception as e:  # profiler unavailable: reported, not fatal
            info["cupti"] = {"error": f"{type(e).__name__}: {e}"[:200]}
        if t.filled is not None:
            m = S.schedule_metrics(t.filled.schedule)
            info["simulated_util"] = m[1] if isinstance(m, tuple) else getattr(m, "utilization", None)
        if dist:
            x = torch.tensor([step, -util], device="cuda")
            dist.all_reduce(x, op=dist.ReduceOp.MAX)
            step, util = float(x[0]), -float(x[1])  # max step time, min util over ranks
        loss = res[-1].loss
        del t
        torch.cuda.empty_cache()
        return step, util, loss, info

    try:
        step_ms, util, loss, info = measure(True)   # measures the cost table first
        plain_ms, plain_util, _, _ = measure(False)  # same schedule costs, K-FAC items dropped
        seqs = cfg.micro_batches * cfg.micro_batch_size * cfg.groups() * (2 if spd == 2 else 1) / spd
        out.update({"step_ms": step_ms, "plain_step_ms": plain_ms, "step_ratio_vs_plain": step_ms / plain_ms,
                    "gpu_util": util, "plain_gpu_util": plain_util,
                    "sequences_per_s": seqs / (step_ms * 1e-3), "loss": loss, **info,
                    "util_definition": "union of F/B/K-FAC/collective op intervals (CUDA events) / cycle wall time, min over ranks; cupti.kernel_util = union of kernel execution intervals (the paper's definition)",
                    "fb": "BERT F/B of every (stage, micro-batch, tape capture) replayed as CUDA graphs (engine graph_fb)"})
        if "measured" in costs_box:
            out["measured_costs"] = costs_box["measured"]
        if world == 1 and t_meas.get("times") is not None:
            # BASELINE configs 2-4 on 2/4/8 B200, SIMULATED by the reference
            # assigner from the item costs measured here (the driver's tiers run
            # one GPU); the 8-GPU row is the north-star Chimera config
            from paper_2211_14133_b200.engine import project_pipeline
            proj = {}
            for n_gpu, sp in sorted(PIPELINE_LADDER.items()):
                if n_gpu == 1:
                    continue
                m = S.parse_method(sp["method"])
                pc = S.PipelineConfig(method=m, stages=sp["stages"], micro_batches=sp["micro_batches"],
                                      micro_batch_size=32, replicas=sp["replicas"],
                                      layers_per_stage=bert.layers // sp["stages"], seq_len=128)
                proj[f"{n_gpu}gpu_{sp['method']}_D{sp['stages']}"] = project_pipeline(t_meas["times"], pc)
            out["projected_from_measured_costs"] = proj
    except Exception as e:  # reported, never fatal for the bench line
        out["error"] = f"{type(e).__name__}: {e}"[:400]
    return out


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-graph", action="store_true", help="eager launches instead of a CUDA graph")
    p.add_argument("--no-pipeline", action="store_true", help="skip the BERT-Large pipeline step section")
    args = p.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if "RANK" not in os.environ:
        world = 1 if args.gpus <= 1 else args.gpus
        if world > 1:
            raise SystemExit("N>1 must be launched with torchrun (one rank per GPU)")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
    else:
        run_gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
