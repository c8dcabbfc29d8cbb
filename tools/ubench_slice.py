"""Slice-kernel bandwidth: pf_slice of a [d x d] fp32 matrix (CUDA-graph
replay, CUDA events).  Bytes = 4 d^2 read + 4 d^2 digit bytes + 12 d written.

    python tools/ubench_slice.py [d ...]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import _lib as L  # noqa: E402
from paper_2211_14133_b200 import kfac as K  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for d in [int(a) for a in sys.argv[1:]] or [1024, 4096, 8192]:
        x = torch.randn(d, d, device="cuda")
        buf = torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda")
        fn = lambda: L.lib().pf_slice(x.data_ptr(), d, d, d, buf.data_ptr(), K._stream())  # noqa: E731
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            with torch.cuda.graph(g):
                for _ in range(10):
                    fn()
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 50
        by = 8.0 * d * d + 12.0 * d
        print(f"d={d:5d}  {us:8.1f} us  {by / us / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
