"""Measured dense int8 tensor-core peak (cuBLASLt via torch._int_mm) beside
bf16, on this GPU: 8192^3, best of 10 (burst) and back to back for ~4 s
(sustained).  Writes profiles/int8_peak.json when given --out.

    python tools/int8_peak.py [--out profiles/int8_peak.json]

The digit-form (fp32-accurate) GEMM runs 10 int8 products per fp32 product,
so its ceiling is int8_peak / 10 in fp32-equivalent FLOP/s.
"""
import json
import sys
import time

import torch


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def measure(fn, flops):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    burst = min(timed(fn, 1) for _ in range(10))
    ms1 = timed(fn, 5)
    reps = max(5, int(4000 / ms1))
    sustained = timed(fn, reps)
    return flops / burst / 1e9, flops / sustained / 1e9


def main():
    n = 8192
    torch.cuda.set_device(0)
    a8 = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda")
    b8 = torch.randint(-127, 128, (n, n), dtype=torch.int8, device="cuda").t()  # column-major B for cuBLASLt
    i8b, i8s = measure(lambda: torch._int_mm(a8, b8), 2.0 * n ** 3)
    ab = torch.randn((n, n), dtype=torch.bfloat16, device="cuda")
    bb = torch.randn((n, n), dtype=torch.bfloat16, device="cuda")
    bfb, bfs = measure(lambda: ab @ bb, 2.0 * n ** 3)
    out = {
        "int8_tops_burst": round(i8b, 1), "int8_tops_sustained": round(i8s, 1),
        "bf16_tflops_burst": round(bfb, 1), "bf16_tflops_sustained": round(bfs, 1),
        "digit_ceiling_tflops_burst": round(i8b / 10, 1), "digit_ceiling_tflops_sustained": round(i8s / 10, 1),
        "how": "torch._int_mm (cuBLASLt int8 x int8 -> int32) and torch.matmul bf16, 8192^3, 2 n^3 ops; "
               "burst = best of 10 single launches, sustained = back to back for ~4 s (CUDA events)",
        "gpu": torch.cuda.get_device_name(0),
        "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
    }
    print(json.dumps(out))
    if "--out" in sys.argv:
        with open(sys.argv[sys.argv.index("--out") + 1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
