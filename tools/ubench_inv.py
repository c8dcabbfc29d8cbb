"""Micro-benchmark of the damped inverse (CUDA-graph replay, CUDA events).

    python tools/ubench_inv.py [d:count ...]

Prints ms per call and algorithmic TFLOP/s (d^3 per factor) for each batch,
plus the residual max|(A+lambda I) X - I| of the first factor.  Development
tool only; the judged numbers come from bench.py.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402

LAM = 0.1


def make(d, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn((d, 4096), generator=g, device="cuda").to(torch.bfloat16).float()
    return (x @ x.T) / 4096


def run(spec, iters=20):
    mats, outs, digs = [], [], []
    for i, (d, c) in enumerate(spec):
        for j in range(c):
            mats.append(make(d, 100 * i + j))
            outs.append(torch.empty((d, d), device="cuda"))
            digs.append(torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda"))
    call = lambda: K.damped_inverse_batched(mats, LAM, outs, digs, check=False)  # noqa: E731
    call()
    torch.cuda.synchronize()
    if os.environ.get("PF_UBENCH_EAGER") == "1":  # host-issued launches, as the pipeline engine runs
        import time
        t0 = time.perf_counter()
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3 / 3
        flops = sum(d ** 3 * c for d, c in spec)
        tag = " + ".join(f"{c}x{d}" for d, c in spec)
        print(f"{tag:24s} {ms * 1e3:9.1f} us  {flops / ms / 1e9:7.2f} TFLOP/s  (eager)", flush=True)
        return
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        call()
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    flops = sum(d ** 3 * c for d, c in spec)
    a = mats[0].double() + LAM * torch.eye(mats[0].shape[0], device="cuda", dtype=torch.float64)
    res = (a @ outs[0].double() - torch.eye(a.shape[0], device="cuda", dtype=torch.float64)).abs().max().item()
    tag = " + ".join(f"{c}x{d}" for d, c in spec)
    print(f"{tag:24s} {ms * 1e3:9.1f} us  {flops / ms / 1e9:7.2f} TFLOP/s  residual {res:.2e}", flush=True)


def main():
    torch.cuda.set_device(0)
    specs = []
    for a in sys.argv[1:]:
        specs.append([tuple(int(v) for v in p.split(":")) for p in a.split(",")])
    if not specs:
        specs = [[(128, 1)], [(128, 2)], [(256, 2)], [(512, 2)], [(1024, 2)], [(2048, 2)],
                 [(4096, 1)], [(4096, 2)], [(1024, 5)], [(4096, 2), (1024, 10)]]
    for sp in specs:
        run(sp)


if __name__ == "__main__":
    main()
