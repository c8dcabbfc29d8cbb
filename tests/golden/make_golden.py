"""Regenerate tests/golden/* from the compiled reference (oracle/_ref).

    make -C oracle && python tests/golden/make_golden.py

schedules.json : reference dumps (build_schedule / enumerate_kfac_works /
                 assign_works) of the hand examples in proj/tests/*.cpp and of
                 the BERT configs 2-4 of BASELINE.json; doubles stored with
                 float.hex() so comparisons are bit-exact.
kfac_small.npz : reference FP64 outputs (curvature_factors, cholesky_spd_inverse,
                 precondition, ngd_step) on SplitMix64 inputs, small sizes.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref as R  # noqa: E402
import helpers as H  # noqa: E402


def named_cases():
    c = {}
    hand = H.hand_costs()
    c["gpipe_d2n2_hand"] = (H.make_config(0, 2, 2), hand, False, 10)
    c["gpipe_d2n2_w2_hand"] = (H.make_config(0, 2, 2, 1, 2), hand, False, 10)
    st = H.hand_costs(); st.t_curv, st.t_inv = 0.1, 0.2
    c["gpipe_d2n2_staleness"] = (H.make_config(0, 2, 2), st, False, 10)
    inf = H.hand_costs(); inf.t_inv = 50.0
    c["gpipe_d2n2_infeasible_cap4"] = (H.make_config(0, 2, 2), inf, False, 4)
    z = H.hand_costs(); z.t_curv = z.t_inv = 0.0
    c["chimera_d2n2_zero_works"] = (H.make_config(2, 2, 2, 2), z, False, 10)
    ip = H.hand_costs(); ip.t_curv, ip.t_inv = 0.05, 0.4
    c["chimera_d4n4_l4_invpar"] = (H.make_config(2, 4, 4, 4), ip, True, 10)
    c["chimera_d4n4_l4_serial"] = (H.make_config(2, 4, 4, 4), ip, False, 10)
    rc = H.hand_costs(); rc.t_b = 2.0
    cfg = H.make_config(1, 4, 8, 2); cfg.recompute = True
    c["1f1b_d4n8_recompute"] = (cfg, rc, False, 10)
    for name, (cfg, costs) in H.bert_configs().items():
        c[name] = (cfg, costs, name != "bert_large_chimera_d8n8", 10)
    return c


def hexify(dump):
    def h(v):
        return v.hex() if isinstance(v, float) else v
    return {
        "header": [h(x) for x in dump.header],
        "items": [[h(x) for x in it] for it in dump.items],
        "staleness": [list(s) for s in dump.staleness],
        "metrics": [h(x) for x in dump.metrics],
        "infeasible": None if dump.infeasible is None else [h(x) for x in dump.infeasible],
        "unplaced": [[h(x) if not isinstance(x, tuple) else list(x) for x in u] for u in dump.unplaced],
    }


def main():
    out = {}
    for name, (cfg, costs, inv_par, cap) in named_cases().items():
        out[name] = {
            "config": {k: int(getattr(cfg, k)) for k in (
                "method", "stages", "micro_batches", "micro_batch_size", "replicas", "devices",
                "layers_per_stage", "seq_len", "recompute")},
            "costs": {k: (getattr(costs, k).hex() if isinstance(getattr(costs, k), float)
                          else getattr(costs, k)) for k in (
                "t_f", "t_b", "t_curv", "t_inv", "t_prec", "m_theta", "m_act", "m_err_peak",
                "m_err_save", "m_curv", "comm_alpha", "comm_beta", "p2p_latency")},
            "inversion_parallel": inv_par,
            "horizon_cap": cap,
            "assign": hexify(R.ref_assign_dump(cfg, costs, inv_par, cap)),
            "build": hexify(R.ref_build_dump(cfg, costs, 2)),
        }
    with open(os.path.join(HERE, "schedules.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)

    # io::trace_to_json of assigned schedules (the trace schema the runtime's
    # measured and simulated timelines are exported in)
    traces = {}
    cases = named_cases()
    for name in ("gpipe_d2n2_hand", "chimera_d4n4_l4_serial", "1f1b_d4n8_recompute"):
        cfg, costs, inv_par, cap = cases[name]
        traces[name] = {"devices_per_group": int(cfg.stages),
                        "trace": json.loads(R.ref_assign_trace(cfg, costs, inv_par, cap, int(cfg.stages)))}
    with open(os.path.join(HERE, "traces.json"), "w") as f:
        json.dump(traces, f, indent=0, sort_keys=True)

    arrays = {}
    for d_in, d_out, n in ((64, 32, 96), (130, 70, 200)):
        a = R.orc_symmetric(1000 + d_in, (d_in, n), 3 ** 0.5)
        e = R.orc_symmetric(2000 + d_out, (d_out, n), 3 ** 0.5)
        A, B = R.ref_curvature_factors(a, e)
        Ai = R.ref_cholesky_spd_inverse(A, 0.1)
        Bi = R.ref_cholesky_spd_inverse(B, 0.1)
        g = R.orc_symmetric(3000 + d_in, (d_out, d_in), 1.0)
        w = R.orc_symmetric(4000 + d_in, (d_out, d_in), 0.02 * 3 ** 0.5)
        P = R.ref_precondition(g, Ai, Bi)
        W, _ = R.ref_ngd_step(w, g, Ai, Bi, 1e-3)
        tag = f"{d_in}x{d_out}x{n}"
        arrays.update({f"{tag}_A": A, f"{tag}_B": B, f"{tag}_Ainv": Ai, f"{tag}_Binv": Bi,
                       f"{tag}_P": P, f"{tag}_W": W})
    np.savez_compressed(os.path.join(HERE, "kfac_small.npz"), **arrays)
    print("wrote", len(out), "schedule goldens and", len(arrays), "arrays")


if __name__ == "__main__":
    main()
