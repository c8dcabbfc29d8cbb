"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference
scheduler, used as an independent checker beside the compiled reference.

Follows, statement for statement in floating point:
  build_schedule       proj/src/schedule.cpp:176-237
  layout_fixed_order   proj/src/schedule.cpp:41-99  (incl. the -1 sentinel quirk)
  layout_chimera       proj/src/schedule.cpp:105-172
  enumerate_kfac_works proj/src/bubblefill.cpp:108-178
  assign_works         proj/src/bubblefill.cpp:180-421
  staleness_report     proj/src/bubblefill.cpp:423-469
Pinned against oracle/_ref (the reference compiled here) by
tests/test_oracle.py; timelines are compared after a canonical sort because
Python's sort is stable and libstdc++'s std::sort is not.
Pure-Python loops: small configurations only.
"""
from __future__ import annotations

import math
from typing import List

EPS = 1e-9
GPIPE, ONEF1B, CHIMERA = 0, 1, 2
FWD, BWD, RECOMP, CURV, INV, PREC, SYNCG, SYNCC = range(8)


def _spd(cfg):
    return 2 if cfg.method == CHIMERA else 1


def _groups(cfg):
    return cfg.replicas // _spd(cfg)


def _devices(cfg):
    return cfg.devices if cfg.devices > 0 else cfg.stages * cfg.replicas // _spd(cfg)


def validate(cfg) -> List[str]:
    v = []
    if cfg.stages < 1: v.append("stages")
    if cfg.micro_batches < 1: v.append("micro_batches")
    if cfg.micro_batch_size < 1: v.append("micro_batch_size")
    if cfg.replicas < 1: v.append("replicas")
    if cfg.layers_per_stage < 1: v.append("layers_per_stage")
    if cfg.seq_len < 1: v.append("seq_len")
    if cfg.method == CHIMERA:
        if cfg.stages % 2: v.append("stages")
        if cfg.micro_batches % 2: v.append("micro_batches")
        if cfg.replicas % 2: v.append("replicas")
    if cfg.stages >= 1 and cfg.replicas >= 1:
        spd = _spd(cfg)
        if (cfg.stages * cfg.replicas) % spd:
            v.append("devices")
        elif cfg.devices > 0 and cfg.devices != cfg.stages * cfg.replicas // spd:
            v.append("devices")
    return v


def _fixed_order(cfg, dur_f, dur_b, p2p):
    D, n = cfg.stages, cfg.micro_batches
    order = []
    for s in range(D):
        seq = []
        if cfg.method == ONEF1B:
            w = min(D - s, n)
            seq += [(False, m) for m in range(w)]
            for m in range(w, n):
                seq += [(True, m - w), (False, m)]
            seq += [(True, m) for m in range(n - w, n)]
        else:
            seq += [(False, m) for m in range(n)] + [(True, m) for m in range(n)]
        order.append(seq)
    f_end = [[-1.0] * n for _ in range(D)]
    b_end = [[-1.0] * n for _ in range(D)]
    free = [0.0] * D
    cur = [0] * D
    tasks, span = [], 0.0
    progressed = True
    while progressed:
        progressed = False
        for s in range(D):
            while cur[s] < len(order[s]):
                bwd, m = order[s][cur[s]]
                if not bwd:
                    ready = 0.0 if s == 0 else f_end[s - 1][m] + p2p
                else:
                    ready = f_end[s][m] if s == D - 1 else b_end[s + 1][m] + p2p
                if ready < 0.0:
                    break
                start = max(ready, free[s])
                dur = dur_b if bwd else dur_f
                (b_end if bwd else f_end)[s][m] = start + dur
                free[s] = start + dur
                tasks.append(dict(pipe=0, round=m, stage=s, bwd=bwd, dev=s, start=start, dur=dur))
                span = max(span, start + dur)
                cur[s] += 1
                progressed = True
    if any(cur[s] != len(order[s]) for s in range(D)):
        raise RuntimeError("pipeline layout deadlocked")
    return tasks, span


def _chimera(cfg, dur_f, dur_b, p2p):
    D, rounds = cfg.stages, cfg.micro_batches // 2
    tasks = []
    for pipe in range(2):
        for r in range(rounds):
            for s in range(D):
                dev = s if pipe == 0 else D - 1 - s
                tasks.append(dict(pipe=pipe, round=r, stage=s, bwd=False, dev=dev, start=-1.0, dur=dur_f))
                tasks.append(dict(pipe=pipe, round=r, stage=s, bwd=True, dev=dev, start=-1.0, dur=dur_b))

    def find(pipe, r, s, bwd):
        return tasks[((pipe * rounds + r) * D + s) * 2 + (1 if bwd else 0)]

    free = [0.0] * D
    span = 0.0
    for _ in range(len(tasks)):
        best, best_start = None, 0.0
        for t in tasks:
            if t["start"] >= 0.0:
                continue
            if not t["bwd"]:
                if t["stage"] == 0:
                    ready = 0.0
                else:
                    dep = find(t["pipe"], t["round"], t["stage"] - 1, False)
                    if dep["start"] < 0.0:
                        continue
                    ready = dep["start"] + dep["dur"] + p2p
            else:
                turn = t["stage"] == D - 1
                dep = find(t["pipe"], t["round"], t["stage"], False) if turn else \
                    find(t["pipe"], t["round"], t["stage"] + 1, True)
                if dep["start"] < 0.0:
                    continue
                ready = dep["start"] + dep["dur"] + (0.0 if turn else p2p)
            start = max(ready, free[t["dev"]])
            key = lambda x: (x["round"], 0 if x["bwd"] else 1, x["pipe"], x["stage"])
            if best is None or start < best_start - EPS:
                best, best_start = t, start
            elif start < best_start + EPS and key(t) < key(best):
                best, best_start = t, start
        if best is None:
            raise RuntimeError("chimera layout deadlocked")
        best["start"] = best_start
        free[best["dev"]] = best_start + best["dur"]
        span = max(span, best_start + best["dur"])
    return tasks, span


def build_schedule(cfg, costs, horizon=1):
    """Returns (timelines, period) with items as tuples
    (dev, kind, stage, micro, layer, factor, start, dur, step)."""
    if validate(cfg) or horizon < 1:
        raise ValueError("invalid config")
    dur_f = costs.t_f
    dur_b = costs.t_b + (costs.t_f if cfg.recompute else 0.0)
    fn = _chimera if cfg.method == CHIMERA else _fixed_order
    tasks, span = fn(cfg, dur_f, dur_b, costs.p2p_latency)
    lines = [[] for _ in range(_devices(cfg))]
    n = cfg.micro_batches
    for step in range(horizon):
        shift = step * span
        for g in range(_groups(cfg)):
            for t in tasks:
                micro = t["round"] if t["pipe"] == 0 else n // 2 + t["round"]
                dev = g * cfg.stages + t["dev"]
                if t["bwd"] and cfg.recompute:
                    lines[dev].append((dev, RECOMP, t["stage"], micro, -1, -1, shift + t["start"], costs.t_f, step))
                    lines[dev].append((dev, BWD, t["stage"], micro, -1, -1, shift + t["start"] + costs.t_f, costs.t_b, step))
                else:
                    lines[dev].append((dev, BWD if t["bwd"] else FWD, t["stage"], micro, -1, -1,
                                       shift + t["start"], t["dur"], step))
    for line in lines:
        line.sort(key=lambda it: it[6])
    return lines, span


def model_collective(nbytes, participants, alpha, beta):
    if nbytes < 0.0 or participants < 2:
        raise ValueError("bad collective")
    return alpha + (nbytes / beta if nbytes > 0.0 else 0.0)


def _replica_devices(cfg, stage):
    out = []
    for g in range(_groups(cfg)):
        out.append(g * cfg.stages + stage)
        if cfg.method == CHIMERA:
            out.append(g * cfg.stages + cfg.stages - 1 - stage)
    return out


def _micros_on(cfg, stage, dev):
    n = cfg.micro_batches
    if cfg.method == CHIMERA:
        down = dev % cfg.stages == stage
        return list(range(0, n // 2) if down else range(n // 2, n))
    return list(range(n))


def enumerate_kfac_works(cfg, costs):
    """List of dicts: kind, stage, layer, factor, micro, device, dur, anchor, preds."""
    if validate(cfg):
        raise ValueError("invalid config")
    layers, w = cfg.layers_per_stage, cfg.replicas
    inv_dur = costs.t_inv / layers
    sync_bytes = float(costs.m_curv) / (2.0 * layers)
    sync_dur = model_collective(sync_bytes, w, costs.comm_alpha, costs.comm_beta) if w > 1 else 0.0
    q = []
    for stage in range(cfg.stages):
        devs = _replica_devices(cfg, stage)
        curv_of = [[] for _ in range(2 * layers)]
        for dev in devs:
            for m in _micros_on(cfg, stage, dev):
                for layer in range(layers):
                    for f in (0, 1):
                        curv_of[2 * layer + f].append(len(q))
                        q.append(dict(kind=CURV, stage=stage, layer=layer, factor=f, micro=m,
                                      device=dev, dur=costs.t_curv, anchor=FWD if f == 0 else BWD,
                                      preds=[]))
        for layer in range(layers):
            for f in (0, 1):
                curvs = curv_of[2 * layer + f]
                sync_idx = -1
                if w > 1:
                    sync_idx = len(q)
                    q.append(dict(kind=SYNCC, stage=stage, layer=layer, factor=f, micro=-1,
                                  device=devs[0], dur=sync_dur, anchor=-1, preds=list(curvs)))
                q.append(dict(kind=INV, stage=stage, layer=layer, factor=f, micro=-1,
                              device=devs[0], dur=inv_dur, anchor=-1,
                              preds=[sync_idx] if sync_idx >= 0 else list(curvs)))
    return q


def _fit(gaps, ready, dur, horizon_end):
    if dur <= 0.0:
        return max(0.0, ready) if ready <= horizon_end + EPS else None
    for b, e in gaps:
        s = max(b, ready)
        if s + dur <= e + EPS:
            return s
    return None


def _occupy(gaps, start, dur):
    if dur <= 0.0:
        return
    for i, (b, e) in enumerate(gaps):
        if start >= b - EPS and start + dur <= e + EPS:
            pieces = []
            if start > b + EPS:
                pieces.append((b, start))
            if start + dur < e - EPS:
                pieces.append((start + dur, e))
            gaps[i:i + 1] = pieces
            return
    raise RuntimeError("occupy() outside any gap")


def _rank(kind):
    return {CURV: 0, SYNCC: 1, INV: 2}.get(kind, 3)


class Infeasible(Exception):
    def __init__(self, unplaced, deficit):
        super().__init__("infeasible")
        self.unplaced = unplaced
        self.deficit = deficit


def assign_works(cfg, costs, inversion_parallel=False, horizon_cap=10):
    """Full pipeline: build base, enumerate, assign.  Returns a dict with
    period, base_period, refresh, prior, timelines (unsorted order irrelevant),
    staleness [(stage, layer, steps)]."""
    base_lines, base_period = build_schedule(cfg, costs, 1)
    queue = enumerate_kfac_works(cfg, costs)
    devices = len(base_lines)
    spd = _spd(cfg)
    step0 = [[it for it in line if it[8] == 0] for line in base_lines]
    anchor = {}
    for d in range(devices):
        for it in step0[d]:
            if it[1] in (FWD, BWD) and it[3] >= 0:
                anchor[(it[1], it[2], it[3], d)] = it[6] + it[7]
    sg = model_collective(float(costs.m_theta), cfg.replicas, costs.comm_alpha,
                          costs.comm_beta) if cfg.replicas > 1 else 0.0
    prec = costs.t_prec / spd
    tail = [[] for _ in range(devices)]
    for d in range(devices):
        last = 0.0
        stage_last = {}
        for it in step0[d]:
            last = max(last, it[6] + it[7])
            if it[1] == BWD:
                stage_last[it[2]] = max(stage_last.get(it[2], 0.0), it[6] + it[7])
        cursor = last
        for end, stage in sorted((e, s) for s, e in stage_last.items()):
            if cfg.replicas > 1:
                tail[d].append((d, SYNCG, stage, -1, -1, -1, cursor, sg, 0))
                cursor += sg
            tail[d].append((d, PREC, stage, -1, -1, -1, cursor, prec, 0))
            cursor += prec
    period = base_period + spd * sg + costs.t_prec
    horizon_end = horizon_cap * period
    gaps = []
    for d in range(devices):
        busy = []
        for k in range(horizon_cap):
            shift = k * period
            for it in step0[d] + tail[d]:
                busy.append((it[6] + shift, (it[6] + it[7]) + shift))
        busy.sort(key=lambda x: x[0])
        g, cursor = [], 0.0
        for b, e in busy:
            if b > cursor + EPS:
                g.append((cursor, b))
            cursor = max(cursor, e)
        if horizon_end > cursor + EPS:
            g.append((cursor, horizon_end))
        gaps.append(g)
    if inversion_parallel and cfg.replicas > 1:
        nxt = {}
        for w in queue:
            if w["kind"] != INV:
                continue
            devs = _replica_devices(cfg, w["stage"])
            k = nxt.get(w["stage"], 0)
            nxt[w["stage"]] = k + 1
            w["device"] = devs[k % len(devs)]
    placed = [False] * len(queue)
    pend = [-1.0] * len(queue)
    out = []
    for _ in range(len(queue)):
        best, best_start = -1, 0.0
        for i, w in enumerate(queue):
            if placed[i]:
                continue
            ready = 0.0
            if w["anchor"] >= 0:
                ready = anchor[(w["anchor"], w["stage"], w["micro"], w["device"])]
            if any(not placed[p] for p in w["preds"]):
                continue
            for p in w["preds"]:
                ready = max(ready, pend[p])
            s = _fit(gaps[w["device"]], ready, w["dur"], horizon_end)
            if s is None:
                continue
            key = (_rank(w["kind"]), w["layer"], w["factor"], w["micro"], w["stage"], w["device"])
            if best < 0 or s < best_start - EPS or (s < best_start + EPS and key < bkey):
                best, best_start, bkey = i, s, key
        if best < 0:
            un = [w for i, w in enumerate(queue) if not placed[i]]
            deficit = 0.0
            for w in un:
                deficit += w["dur"]
            raise Infeasible(un, deficit)
        w = queue[best]
        _occupy(gaps[w["device"]], best_start, w["dur"])
        placed[best] = True
        pend[best] = best_start + w["dur"]
        out.append((w["device"], w["kind"], w["stage"], w["micro"], w["layer"], w["factor"],
                    best_start, w["dur"]))
    step_eps = EPS * max(1.0, period)

    def step_of_end(e):
        if period <= 0.0:
            return 1
        return max(1, int(math.ceil((e - step_eps) / period)))

    refresh = 1
    for it in out:
        refresh = max(refresh, step_of_end(it[6] + it[7]))
    lines = [[] for _ in range(devices)]
    for d in range(devices):
        for k in range(refresh):
            shift = k * period
            for it in step0[d] + tail[d]:
                lines[d].append(it[:6] + (it[6] + shift, it[7], k))
    for it in out:
        lines[it[0]].append(it + (step_of_end(it[6] + it[7]) - 1,))
    for line in lines:
        line.sort(key=lambda x: (x[6], x[1]))
    # staleness (bubblefill.cpp:423-469)
    cycle = refresh * period
    prec_start, inv_end = {}, {}
    for line in lines:
        for it in line:
            if it[1] == PREC:
                k = (it[2], it[8])
                prec_start[k] = min(prec_start.get(k, it[6]), it[6])
            elif it[1] == INV:
                inv_end[(it[2], max(it[4], 0), 1 if it[5] == 1 else 0)] = it[6] + it[7]
    per_layer = {}
    for (stage, layer, _f), end in sorted(inv_end.items()):
        uses = refresh
        if cycle > 0.0:
            uses = 0
            for k in range(2 * refresh):
                ps = prec_start.get((stage, k % refresh))
                if ps is None:
                    continue
                start = ps + (k // refresh) * cycle
                if start >= end - EPS and start < end + cycle - EPS:
                    uses += 1
            uses = max(uses, 1)
        per_layer[(stage, layer)] = max(per_layer.get((stage, layer), uses), uses)
    stale = [(s, l, v) for (s, l), v in sorted(per_layer.items())]
    last_inv = {}
    for line in lines:
        for it in line:
            if it[1] == INV:
                last_inv[it[2]] = max(last_inv.get(it[2], it[6] + it[7]), it[6] + it[7])
    prior = 0
    for line in lines:
        for it in line:
            if it[1] == PREC and it[2] in last_inv and it[6] < last_inv[it[2]] - EPS:
                prior += 1
    return dict(period=period, base_period=base_period, refresh=refresh, prior=prior,
                lines=lines, staleness=stale)
