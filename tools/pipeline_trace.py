"""Measured-timeline trace: run one recorded PipeFisher cycle
of BERT-Large on this GPU and write it in the reference trace schema
(proj/src/io/trace.cpp:38-63), beside the SIMULATED schedule of BASELINE
config 3 (Chimera D=8) built by the reference assigner from the costs
measured in the same run.

    python tools/pipeline_trace.py OUT_DIR

Writes OUT_DIR/pipeline_trace_measured.json and
OUT_DIR/pipeline_trace_simulated_chimera_d8.json (chrome://tracing / Perfetto).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import schedule as S  # noqa: E402
from paper_2211_14133_b200.bert import BertConfig  # noqa: E402
from paper_2211_14133_b200.engine import (PipeFisherTrainer, costs_from_times, measured_trace,  # noqa: E402
                                          project_pipeline, schedule_trace, MeasuredTimes)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
    os.makedirs(out, exist_ok=True)
    torch.cuda.set_device(0)
    bert = BertConfig.large()
    cfg = S.PipelineConfig(method=S.Method.GPipe, stages=1, micro_batches=4, micro_batch_size=32, replicas=1,
                           layers_per_stage=bert.layers, seq_len=128)
    t = PipeFisherTrainer(cfg, bert, kfac=True, refresh=2, costs="measured", seed=11)
    t.run_cycle()
    r = t.run_cycle(record=True)
    doc = measured_trace(t)
    doc["otherData"].update({"config": "BERT-Large, D=1 (inline K-FAC), 4 micro-batches of 32x128",
                             "step_ms": r.step_ms, "util_union": r.util})
    with open(os.path.join(out, "pipeline_trace_measured.json"), "w") as f:
        json.dump(doc, f, indent=1)
    m = t.measured
    c8 = S.PipelineConfig(method=S.Method.Chimera, stages=8, micro_batches=8, micro_batch_size=32, replicas=2,
                          layers_per_stage=3, seq_len=128)
    proj = project_pipeline(m, c8)
    per = lambda v: v / m.layers * 3  # noqa: E731
    costs = costs_from_times(MeasuredTimes(f=per(m.f), b=per(m.b), curv=m.curv, inv=m.inv, prec=per(m.prec),
                                           layers=3, stages_per_device=2, param_bytes=int(per(m.param_bytes)),
                                           factor_bytes=int(per(m.factor_bytes))))
    filled = S.assign_works(S.build_schedule(c8, costs), c8, costs, S.enumerate_kfac_works(c8, costs),
                            S.AssignOptions())
    sim = schedule_trace(filled.schedule, 8)
    sim["otherData"] = {"source": "simulated by assign_works from the item costs measured on this GPU",
                        **{k: v for k, v in proj.items() if k != "cost_table"}}
    with open(os.path.join(out, "pipeline_trace_simulated_chimera_d8.json"), "w") as f:
        json.dump(sim, f, indent=1)
    print(json.dumps({"measured_events": len(doc["traceEvents"]), "measured": doc["otherData"],
                      "simulated_events": len(sim["traceEvents"]), "simulated": sim["otherData"]}, indent=1))


if __name__ == "__main__":
    main()
