"""SYRK micro-benchmark: feature-major [d x n] vs token-major [n x d] tapes
(CUDA-graph replay, CUDA events), single factors and the bench's grouped
12-factor BERT-Large launch.  Development tool."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402


def timed(fn, iters=20):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    # PF_UB_PER_GRAPH=n: n calls captured back to back in one graph (no
    # per-graph launch gap between them); default 1 call per graph
    per = int(os.environ.get("PF_UB_PER_GRAPH", "1"))
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters / per


def main():
    torch.cuda.set_device(0)
    cases = [[(128, 64)], [(128, 512)], [(128, 4096)], [(256, 4096)], [(512, 4096)], [(1024, 4096)], [(2048, 4096)], [(4096, 4096)],
             [(1024, 4096)] * 10 + [(4096, 4096)] * 2]
    for spec in cases:
        xs_f = [torch.randn((d, n), device="cuda").to(torch.bfloat16) for d, n in spec]
        xs_t = [x.t().contiguous() for x in xs_f]
        fs = [torch.empty((d, d), device="cuda") for d, _ in spec]
        flops = sum(d * (d + 1) * n for d, n in spec)
        t_f = timed(lambda: K.syrk([(x, f, 1.0, False) for x, f in zip(xs_f, fs)], fill_upper=False))
        t_t = timed(lambda: K.syrk([(x, f, 1.0, False, True) for x, f in zip(xs_t, fs)], fill_upper=False))
        tag = " + ".join(f"{spec.count(c)}x{c[0]}" for c in dict.fromkeys(spec))
        print(f"{tag:24s} feature-major {t_f * 1e3:8.1f} us {flops / t_f / 1e9:7.1f} TF/s   "
              f"token-major {t_t * 1e3:8.1f} us {flops / t_t / 1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
