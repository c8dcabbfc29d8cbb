"""Bit-exact parity of the B200 host scheduler (csrc/host/*.cpp through the
C-ABI) with the reference scheduler (oracle/_ref, the unmodified
/root/reference sources compiled here) and with the committed goldens.

Mirrors the reference's own suites: proj/tests/test_schedule.cpp,
proj/tests/test_bubblefill.cpp and the acceptance criteria 1-4
(proj/tests/acceptance.cpp).  "Bit-exact" = every double equal and the
per-device item order identical.
"""
import json
import math
import os

import pytest

from paper_2211_14133_b200 import schedule as S
from oracle import ref as R

import helpers as H

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "schedules.json")
need_ref = pytest.mark.skipif(not R.ref_available(), reason="oracle/_ref not built")


def product_assign(cfg, costs, inv_par=False, cap=10):
    base = S.build_schedule(cfg, costs, 1)
    q = S.enumerate_kfac_works(cfg, costs)
    return S.assign_works(base, cfg, costs, q, S.AssignOptions(inv_par, cap))


def compare_assign(cfg, costs, inv_par=False, cap=10):
    want = R.ref_assign_dump(cfg, costs, inv_par, cap)
    try:
        got = product_assign(cfg, costs, inv_par, cap)
    except S.InfeasibleError as e:
        assert want.infeasible is not None, "product infeasible, reference feasible"
        assert e.deficit_ms == want.infeasible[0]
        assert len(e.unplaced) == want.infeasible[1]
        assert str(e) == want.infeasible[2]
        assert [(int(w.kind), w.stage, w.layer, int(w.factor),
                 -1 if w.micro_batch is None else w.micro_batch, w.device, w.duration)
                for w in e.unplaced] == [u[:7] for u in want.unplaced]
        return None
    assert want.infeasible is None, "reference infeasible, product feasible"
    assert (got.schedule.period, got.base_period, got.refresh_period,
            got.preconditions_using_prior_inverses, got.schedule.device_count()) == want.header
    assert H.items_of(got.schedule) == want.items  # exact order, exact doubles
    assert [(e.stage, e.layer, e.staleness_steps) for e in got.staleness] == want.staleness
    span, util, _ = S.schedule_metrics(got.schedule)
    assert (span, util) == want.metrics
    return got


# ---------------------------------------------------------------- build_schedule
@need_ref
@pytest.mark.parametrize("method", [0, 1, 2])
@pytest.mark.parametrize("depth", [2, 4, 8])
@pytest.mark.parametrize("factor", [1, 2, 3])
@pytest.mark.parametrize("costs", [(1.0, 1.0, 0.0), (0.37, 0.37, 0.0), (1.25, 2.5, 0.0),
                                   (1.0, 2.0, 0.25), (1.0, 1.0, 1.0), (1.0, 1.5, 1.5)])
def test_build_schedule_matches_reference(method, depth, factor, costs):
    cfg = H.make_config(method, depth, depth * factor)
    t = S.CostTable(t_f=costs[0], t_b=costs[1], p2p_latency=costs[2])
    got = S.build_schedule(cfg, t, 2)
    want = R.ref_build_dump(cfg, t, 2)
    assert (got.period, got.horizon_steps, got.refresh_period, got.device_count()) == want.header
    assert H.items_of(got) == want.items
    idle, totals = S.extract_bubbles(got)
    mine = []
    for d, (gaps, tot) in enumerate(zip(idle, totals)):
        mine.append(("T", d, tot))
        mine += [("G", d, g.begin, g.end) for g in gaps]
    assert mine == want.bubbles
    span, util, _ = S.schedule_metrics(got)
    assert (span, util) == want.metrics
    assert [f"{a}: {b}" for a, b in S.validate_schedule(got, cfg)] == want.violations


@need_ref
@pytest.mark.parametrize("method", [0, 1])
def test_recompute_and_replicas_match_reference(method):
    for replicas in (1, 2, 3):
        cfg = H.make_config(method, 4, 8, 2, replicas)
        cfg.recompute = True
        t = S.CostTable(t_f=0.7, t_b=1.3, p2p_latency=0.05)
        got = S.build_schedule(cfg, t, 3)
        assert H.items_of(got) == R.ref_build_dump(cfg, t, 3).items


def test_gpipe_d2n2_hand_simulation():
    """proj/tests/test_schedule.cpp:44-67."""
    s = S.build_schedule(H.make_config(0, 2, 2), S.CostTable(t_f=1.0, t_b=1.0))
    assert s.makespan() == 6.0
    starts = {(w.kind, w.micro_batch): w.start for w in s.timelines[0]}
    assert starts[(S.WorkKind.Forward, 0)] == 0.0 and starts[(S.WorkKind.Forward, 1)] == 1.0
    assert starts[(S.WorkKind.Backward, 0)] == 4.0 and starts[(S.WorkKind.Backward, 1)] == 5.0
    idle, _ = S.extract_bubbles(s)
    assert [(g.begin, g.end) for g in idle[0]] == [(2.0, 4.0)]
    assert [(g.begin, g.end) for g in idle[1]] == [(0.0, 1.0), (5.0, 6.0)]


def test_chimera_d4n4_slot_table():
    """proj/tests/test_schedule.cpp:77-117 (32-slot expected table)."""
    s = S.build_schedule(H.make_config(2, 4, 4), S.CostTable(t_f=1.0, t_b=1.0))
    assert s.makespan() == 10.0
    assert abs(S.schedule_metrics(s)[1] - 0.8) < 1e-12
    F, B = S.WorkKind.Forward, S.WorkKind.Backward
    expect = [
        [(F, 0, 0, 0), (F, 0, 1, 1), (F, 3, 2, 3), (B, 3, 2, 4), (F, 3, 3, 5), (B, 3, 3, 6),
         (B, 0, 0, 7), (B, 0, 1, 9)],
        [(F, 1, 0, 1), (F, 2, 2, 2), (F, 1, 1, 3), (F, 2, 3, 4), (B, 2, 2, 5), (B, 1, 0, 6),
         (B, 2, 3, 7), (B, 1, 1, 8)],
        [(F, 2, 0, 2), (F, 1, 2, 1), (F, 2, 1, 4), (F, 1, 3, 3), (B, 2, 0, 5), (B, 1, 2, 6),
         (B, 2, 1, 7), (B, 1, 3, 8)],
        [(F, 3, 0, 3), (F, 0, 2, 0), (F, 3, 1, 5), (F, 0, 3, 1), (B, 3, 0, 4), (B, 0, 2, 7),
         (B, 3, 1, 6), (B, 0, 3, 9)],
    ]
    for d, slots in enumerate(expect):
        got = {(w.kind, w.stage, w.micro_batch): w.start for w in s.timelines[d]}
        for kind, stage, micro, start in slots:
            assert got[(kind, stage, micro)] == start


def test_chimera_d2n2_has_no_bubbles():
    s = S.build_schedule(H.make_config(2, 2, 2), S.CostTable(t_f=1.0, t_b=1.0))
    idle, _ = S.extract_bubbles(s)
    assert all(not g for g in idle)
    assert s.makespan() == 4.0


def test_utilization_values():
    """acceptance criterion 2 (acceptance.cpp:82-92)."""
    unit = S.CostTable(t_f=1.0, t_b=1.0)
    assert abs(S.schedule_metrics(S.build_schedule(H.make_config(0, 4, 4), unit))[1] - 4 / 7) < 1e-12
    assert abs(S.schedule_metrics(S.build_schedule(H.make_config(2, 4, 4), unit))[1] - 0.8) < 1e-12


@pytest.mark.parametrize("method", [0, 1, 2])
@pytest.mark.parametrize("depth", [2, 4, 8])
def test_makespan_equals_critical_path(method, depth):
    """acceptance criterion 1: makespan = C_f T_f + C_b T_b at N = D, with
    C_f = C_b = 2D-1 for GPipe/1F1B and C_f = D, C_b = 2D-2 for Chimera."""
    cf, cb = (depth, 2 * depth - 2) if method == 2 else (2 * depth - 1, 2 * depth - 1)
    for unit in (1.0, 0.37):
        s = S.build_schedule(H.make_config(method, depth, depth), S.CostTable(t_f=unit, t_b=unit))
        assert s.makespan() == pytest.approx(cf * unit + cb * unit, rel=1e-12)
        idle, totals = S.extract_bubbles(s)
        # every device idles exactly the formula bubble
        busy = S.schedule_metrics(s)[2]
        assert all(abs(t - (s.makespan() - b)) < 1e-9 for t, b in zip(totals, busy))


def test_invalid_config_raises():
    with pytest.raises(ValueError, match="invalid config"):
        S.build_schedule(H.make_config(2, 3, 4), S.CostTable(t_f=1, t_b=1))
    with pytest.raises(ValueError):
        S.build_schedule(H.make_config(0, 2, 2), S.CostTable(t_f=1, t_b=1), 0)
    v = S.validate_config(S.PipelineConfig(method=S.Method.Chimera, stages=3, micro_batches=3,
                                           replicas=1))
    assert ("stages", "Chimera requires D even") in v
    assert ("replicas", "Chimera requires W even") in v


# ---------------------------------------------------------------- assignment
@need_ref
def test_hand_example_gpipe_d2n2():
    """proj/tests/test_bubblefill.cpp:227-267."""
    f = compare_assign(H.make_config(0, 2, 2), H.hand_costs())
    placed = {(w.kind, w.stage, w.factor, w.micro_batch): w for line in f.schedule.timelines
              for w in line if w.kind in (S.WorkKind.Curvature, S.WorkKind.Inversion)}
    ca0 = placed[(S.WorkKind.Curvature, 0, S.Factor.A, 0)]
    ca1 = placed[(S.WorkKind.Curvature, 0, S.Factor.A, 1)]
    ia = placed[(S.WorkKind.Inversion, 0, S.Factor.A, None)]
    assert (ca0.start, ca0.end(), ca1.start, ca1.end(), ia.start, ia.end()) == (2.0, 2.5, 2.5, 3.0, 3.0, 4.0)
    assert f.schedule.period == 6.25
    assert placed[(S.WorkKind.Curvature, 0, S.Factor.B, 0)].start == pytest.approx(6.25 + 2.0)
    assert placed[(S.WorkKind.Inversion, 0, S.Factor.B, None)].end() == pytest.approx(6.25 + 4.0)
    assert f.refresh_period == 3
    assert all(e.staleness_steps == 3 for e in f.staleness)


@need_ref
def test_named_cases_match_reference():
    for name, rec in json.load(open(GOLDEN)).items():
        cfg, costs = _golden_cfg(rec)
        compare_assign(cfg, costs, rec["inversion_parallel"], rec["horizon_cap"])


def _golden_cfg(rec):
    cfg = S.PipelineConfig(**{k: (S.Method(v) if k == "method" else
                                  bool(v) if k == "recompute" else v)
                              for k, v in rec["config"].items()})
    costs = S.CostTable(**{k: (float.fromhex(v) if isinstance(v, str) else v)
                           for k, v in rec["costs"].items()})
    return cfg, costs


def _unhex(x):
    return float.fromhex(x) if isinstance(x, str) else x


def test_named_cases_match_committed_goldens():
    """Runs without oracle/_ref: the goldens were produced by the reference."""
    for name, rec in json.load(open(GOLDEN)).items():
        cfg, costs = _golden_cfg(rec)
        want = rec["assign"]
        try:
            got = product_assign(cfg, costs, rec["inversion_parallel"], rec["horizon_cap"])
        except S.InfeasibleError as e:
            assert want["infeasible"] is not None, name
            assert e.deficit_ms == _unhex(want["infeasible"][0])
            assert len(e.unplaced) == want["infeasible"][1]
            continue
        assert want["infeasible"] is None, name
        assert list(H.items_of(got.schedule)) == [tuple(_unhex(x) for x in it) for it in want["items"]], name
        assert [got.schedule.period, got.base_period, got.refresh_period,
                got.preconditions_using_prior_inverses, got.schedule.device_count()] == \
            [_unhex(x) for x in want["header"]], name
        bwant = rec["build"]
        b = S.build_schedule(cfg, costs, 2)
        assert list(H.items_of(b)) == [tuple(_unhex(x) for x in it) for it in bwant["items"]], name


@need_ref
def test_acceptance_seed_1618_200_tables():
    """acceptance.cpp:205-253: 200 seeded tables, incl. W=4 and inversion parallelism."""
    rng = H.SplitMix64(1618)
    feasible = 0
    for _ in range(200):
        cfg, costs, inv_par = H.acceptance_table(rng)
        got = compare_assign(cfg, costs, inv_par, 10)
        if got is not None:
            feasible += 1
            assert got.refresh_period <= 10
            assert got.schedule.period - S.build_schedule(cfg, costs).period == pytest.approx(costs.t_prec, abs=1e-9)
    assert feasible >= 20


@need_ref
def test_soundness_seed_271828():
    rng = H.SplitMix64(271828)
    for _ in range(25):
        cfg, costs = H.soundness_table(rng)
        compare_assign(cfg, costs)


@need_ref
def test_monotone_seed_577215_and_nonfree_comm():
    """test_bubblefill.cpp:363-390 + non-free communication / W>1 variants."""
    rng = H.SplitMix64(577215)
    for _ in range(15):
        method = [0, 1][rng.next() % 2]
        depth = 2 + rng.next() % 3
        cfg = H.make_config(method, depth, depth, 1 + rng.next() % 2)
        costs = S.CostTable(t_f=1.0, t_b=1.0, t_curv=2.0 * rng.uniform(), t_inv=2.0 * rng.uniform(),
                            t_prec=rng.uniform())
        compare_assign(cfg, costs)
        larger = S.CostTable(**{**costs.__dict__, "t_f": 2.0, "t_b": 2.0})
        compare_assign(cfg, larger)
    rng = H.SplitMix64(4242)
    for _ in range(40):
        method = [0, 1, 2][rng.next() % 3]
        depth = 2 + 2 * (rng.next() % 3) if method == 2 else 2 + rng.next() % 4
        cfg = H.make_config(method, depth, depth * (1 + rng.next() % 2), 1 + rng.next() % 3,
                            (2 if method == 2 else 1) * (1 + rng.next() % 2))
        costs = S.CostTable(t_f=1.0, t_b=0.5 + 2 * rng.uniform(), t_curv=rng.uniform(),
                            t_inv=3 * rng.uniform(), t_prec=rng.uniform(),
                            m_theta=int(1e6 * rng.uniform()), m_curv=int(4e6 * rng.uniform()),
                            comm_alpha=0.05 * rng.uniform(), comm_beta=1e6 + 1e7 * rng.uniform(),
                            p2p_latency=0.2 * rng.uniform())
        compare_assign(cfg, costs, bool(rng.next() % 2), 10)


@need_ref
@pytest.mark.parametrize("p2p", [0.5, 0.99, 1.0, 1.5])
def test_p2p_sentinel_quirk_reproduced(p2p):
    """p2p >= 1 ms breaks the reference's -1 sentinel; parity
    includes the quirk (makespans 7.0, 7.98, 6.0, 6.5 for GPipe D2N2)."""
    cfg = H.make_config(0, 2, 2)
    t = S.CostTable(t_f=1.0, t_b=1.0, p2p_latency=p2p)
    got = S.build_schedule(cfg, t)
    assert H.items_of(got) == R.ref_build_dump(cfg, t).items
    assert got.makespan() == {0.5: 7.0, 0.99: 7.98, 1.0: 6.0, 1.5: 6.5}[p2p]


@need_ref
@pytest.mark.parametrize("name", list(H.bert_configs()))
@pytest.mark.parametrize("inv_par", [False, True])
def test_bert_configs_match_reference(name, inv_par):
    cfg, costs = H.bert_configs()[name]
    compare_assign(cfg, costs, inv_par, 10)


def test_queue_counts_and_durations():
    """test_bubblefill.cpp:190-225."""
    costs = H.hand_costs()
    q = S.enumerate_kfac_works(H.make_config(0, 2, 4, 3), costs)
    for s in range(2):
        kinds = [w.kind for w in q.items if w.stage == s]
        assert kinds.count(S.WorkKind.Curvature) == 24
        assert kinds.count(S.WorkKind.Inversion) == 6
        assert kinds.count(S.WorkKind.SyncCurvature) == 0
    q = S.enumerate_kfac_works(H.make_config(0, 2, 4, 3, 2), costs)
    kinds = [w.kind for w in q.items if w.stage == 0]
    assert (kinds.count(S.WorkKind.SyncCurvature), kinds.count(S.WorkKind.Curvature),
            kinds.count(S.WorkKind.Inversion)) == (6, 48, 6)
    q = S.enumerate_kfac_works(H.make_config(0, 2, 4, 4), costs)
    for w in q.items:
        if w.kind == S.WorkKind.Inversion:
            assert w.duration == costs.t_inv / 4.0


@need_ref
def test_queue_matches_reference():
    for cfg, costs in [(H.make_config(2, 4, 8, 3, 4), H.hand_costs()),
                       (H.make_config(1, 4, 4, 6, 2), H.bert_configs()["bert_large_1f1b_d4n4w2"][1])]:
        q = S.enumerate_kfac_works(cfg, costs)
        want = R.ref_queue_dump(cfg, costs).queue
        got = [(int(w.kind), w.stage, w.layer, int(w.factor),
                -1 if w.micro_batch is None else w.micro_batch, w.device, w.duration,
                -1 if w.base_anchor is None else int(w.base_anchor), tuple(w.preds)) for w in q.items]
        assert got == want


def test_infeasible_payload():
    """test_bubblefill.cpp:392-408."""
    costs = H.hand_costs()
    costs.t_inv = 50.0
    with pytest.raises(S.InfeasibleError) as e:
        product_assign(H.make_config(0, 2, 2), costs, False, 4)
    assert len(e.value.unplaced) == 4
    assert all(w.kind == S.WorkKind.Inversion for w in e.value.unplaced)
    assert e.value.deficit_ms == pytest.approx(200.0)


def test_collective_model():
    assert S.model_collective(12345678.0, 4, 0.0, math.inf) == 0.0
    assert S.model_collective(0.0, 2, 0.1, 1e6) == pytest.approx(0.1)
    assert S.model_collective(1e6, 2, 0.0, 1e6) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        S.model_collective(1.0, 1, 0.0, 1.0)
    with pytest.raises(ValueError):
        S.model_collective(-1.0, 2, 0.0, 1.0)


def test_empty_queue_and_zero_costs():
    cfg = H.make_config(0, 2, 2)
    costs = H.hand_costs()
    base = S.build_schedule(cfg, costs)
    f = S.assign_works(base, cfg, costs, S.KfacWorkQueue())
    assert f.refresh_period == 1
    kinds = [w.kind for line in f.schedule.timelines for w in line]
    assert kinds.count(S.WorkKind.Precondition) == 2
    zero = S.CostTable()
    f = product_assign(cfg, zero)
    assert f.refresh_period == 1
    assert all(e.staleness_steps == 1 for e in f.staleness)


def test_inversion_parallel_spreads_devices():
    cfg = H.make_config(2, 4, 4, 4)
    costs = H.hand_costs()
    costs.t_curv, costs.t_inv = 0.05, 0.4
    for inv_par, ndev in ((True, 2), (False, 1)):
        f = product_assign(cfg, costs, inv_par)
        per_stage = {}
        for line in f.schedule.timelines:
            for w in line:
                if w.kind == S.WorkKind.Inversion:
                    per_stage.setdefault(w.stage, set()).add(w.device)
        assert all(len(v) == ndev for v in per_stage.values())


def test_custom_queue_with_measured_durations():
    """Per-item durations are read from the queue (bubblefill.cpp:317)."""
    cfg = H.make_config(0, 4, 4, 2)
    costs = H.hand_costs()
    base = S.build_schedule(cfg, costs)
    q = S.enumerate_kfac_works(cfg, costs)
    for i, w in enumerate(q.items):
        w.duration = 0.01 * (1 + i % 7)
    f = S.assign_works(base, cfg, costs, q)
    placed = [w for line in f.schedule.timelines for w in line
              if w.kind in (S.WorkKind.Curvature, S.WorkKind.Inversion)]
    assert len(placed) == len(q.items)
    assert sorted(w.duration for w in placed) == sorted(w.duration for w in q.items)


def _canon_events(doc):
    return sorted(doc["traceEvents"], key=lambda e: (e["tid"], e["ts"], e["name"], e["dur"]))


@pytest.mark.parametrize("name", ["gpipe_d2n2_hand", "chimera_d4n4_l4_serial", "1f1b_d4n8_recompute"])
def test_schedule_trace_matches_reference_trace_to_json(name):
    """engine.schedule_trace == the reference's io::trace_to_json
    (proj/src/io/trace.cpp:38-63) on the same assigned schedule: event names,
    ts/dur in us (llround), pid/tid, args — compared after a canonical order
    (the reference's final std::sort is unstable on ties).  Golden: the
    compiled reference (tests/golden/make_golden.py)."""
    from paper_2211_14133_b200.engine import schedule_trace
    here = os.path.join(os.path.dirname(__file__), "golden")
    gold = json.load(open(os.path.join(here, "traces.json")))[name]
    g = json.load(open(GOLDEN))[name]
    cfg = S.PipelineConfig(method=S.Method(g["config"]["method"]), stages=g["config"]["stages"],
                           micro_batches=g["config"]["micro_batches"],
                           micro_batch_size=g["config"]["micro_batch_size"], replicas=g["config"]["replicas"],
                           devices=g["config"]["devices"], layers_per_stage=g["config"]["layers_per_stage"],
                           seq_len=g["config"]["seq_len"], recompute=bool(g["config"]["recompute"]))
    costs = S.CostTable(**{k: (float.fromhex(v) if isinstance(v, str) else v) for k, v in g["costs"].items()})
    filled = product_assign(cfg, costs, g["inversion_parallel"], g["horizon_cap"])
    ours = schedule_trace(filled.schedule, gold["devices_per_group"])
    assert _canon_events(ours) == _canon_events(gold["trace"])
