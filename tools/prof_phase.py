"""Run one phase of bench.py's layer step in a loop, for ncu captures.

    python tools/prof_phase.py {curvature|inversion|precondition|step} [iters]

The same device state and calls as bench.py (LayerStep), nothing timed here:
numbers printed under a profiler are never bench values.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2211_14133_b200 import kfac as K  # noqa: E402


def main():
    phase = sys.argv[1] if len(sys.argv) > 1 else "curvature"
    iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    torch.cuda.set_device(0)
    st = bench.LayerStep(torch, K, seed=1234)
    st.curvature()
    st.invert()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: setup is not captured
    for _ in range(iters):
        if phase in ("curvature", "step"):
            st.curvature()
        if phase in ("inversion", "step"):
            st.invert()
        if phase in ("precondition", "step"):
            st.precondition()
    torch.cuda.synchronize()
    print("done", phase, iters, "launches", K.kernel_launches())


if __name__ == "__main__":
    main()
