"""Per-launch cost of the small kernels on the inversion chain, inside a CUDA
graph (CUDA events around R back-to-back replays of K chained calls):

  slice      pf_slice of a 128 x 128 fp32 block        (1 launch)
  precond    pf_precondition 128 x 128                 (3 slices, GEMM, slice, GEMM)

Development tool only.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402


def graph_time(fn, chain=50, reps=10):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(chain):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * chain)


def main():
    torch.cuda.set_device(0)
    for d in (128, 256, 512):
        x = torch.randn(d, d, device="cuda")
        sm = K.slice_matrix(x)
        t_slice = graph_time(lambda: K.L.lib().pf_slice(x.data_ptr(), d, d, d, sm.digits.data_ptr(), K._stream()))
        a = torch.eye(d, device="cuda") + 0.01 * torch.randn(d, d, device="cuda")
        g = torch.randn(d, d, device="cuda")
        out = torch.empty_like(g)
        t_prec = graph_time(lambda: K.L.lib().pf_precondition(
            a.data_ptr(), g.data_ptr(), a.data_ptr(), out.data_ptr(), d, d,
            K._WS.get(K.precondition_workspace_bytes(d, d), g.device, "prec").data_ptr(),
            K.precondition_workspace_bytes(d, d), K._stream()))
        print(f"d={d:4d}  slice {t_slice:6.2f} us   precondition {t_prec:6.2f} us  "
              f"=> gemm ~ {(t_prec - 4 * t_slice) / 2:6.2f} us", flush=True)


if __name__ == "__main__":
    main()
