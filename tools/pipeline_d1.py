"""D = 1 BERT-Large PipeFisher step vs the plain step, with the CUPTI
kernel-activity breakdown (engine.kernel_activity): where the inline K-FAC
block's time goes (K-FAC kernels, other kernels, idle).  Development tool."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import schedule as S  # noqa: E402
from paper_2211_14133_b200.bert import BertConfig  # noqa: E402
from paper_2211_14133_b200.engine import PipeFisherTrainer, kernel_activity  # noqa: E402


def main():
    torch.cuda.set_device(0)
    bert = BertConfig.large()
    cfg = S.PipelineConfig(method=S.Method.GPipe, stages=1, micro_batches=4, micro_batch_size=32,
                           replicas=1, layers_per_stage=24, seq_len=128,
                           recompute=os.environ.get("PF_RECOMPUTE") == "1")
    out = {}
    for kfac in (True, False):
        t = PipeFisherTrainer(cfg, bert, kfac=kfac, refresh=2, seed=11,
                              graph_fb=os.environ.get("PF_GRAPH_FB") == "1")
        t.run_cycle()
        t.run_cycle()  # the second call of a batched inversion captures its graph
        walls, steps = [], []
        for _ in range(3):
            w0 = time.perf_counter()
            r = t.run_cycle()
            walls.append((time.perf_counter() - w0) * 1e3 / t.refresh)
            steps.append(r.step_ms)
        r = t.run_cycle(record=True)
        kinds = {}
        for kind, a, b, m in getattr(t, "last_trace", []):
            kinds.setdefault(kind, [0, 0.0])
            kinds[kind][0] += 1
            kinds[kind][1] += b - a
        out["kfac" if kfac else "plain"] = {"step_ms": sum(steps) / 3, "host_wall_ms_per_step": sum(walls) / 3,
                                            "op_ms_per_cycle": {k: {"ops": v[0], "ms": round(v[1], 3)} for k, v in kinds.items()},
                                            "cycle_ms": r.step_ms * t.refresh,
                                            "cupti": kernel_activity(t)}
        if os.environ.get("PF_D1_TRACE") == "1":  # the recorded cycle's op intervals (ms from cycle start)
            out["kfac" if kfac else "plain"]["trace"] = [(k, round(a, 2), round(b, 2), m.get("step"))
                                                         for k, a, b, m in getattr(t, "last_trace", [])]
        del t
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
