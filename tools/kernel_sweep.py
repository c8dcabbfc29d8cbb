"""K-FAC kernel sweep (BASELINE.json configs[4]): factor dim d in
{256 ... 8192}, n = 4096 tokens, each kernel timed with CUDA events around
CUDA-graph replays (inputs resident, L2 > working set only for small d).

  curvature SYRK      d(d+1)n FLOP, bytes 2dn + 2d(d+1) (bf16 tape in, fp32 lower out)
  damped inverse      d^3 FLOP (one factor = latency; 8 factors = throughput)
  precondition+update 2d^3 + 2d^3 FLOP (d_out = d_in = d)

Prints one JSON object per row and a markdown table; roofline denominators
from MEASURED_PEAKS.json (bf16 dense sustained, HBM copy) and the int8-digit
fp32-accurate ceiling 2 x bf16 / 10.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402

N = 4096


def peaks():
    """Burst peaks (kernels here are timed alone): bf16 dense and HBM copy
    from MEASURED_PEAKS.json, int8 dense from profiles/int8_peak.json (the
    digit-form ceiling is int8 / 10)."""
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bf16, hbm, src = p["bf16_tflops"], p["hbm_gbs"], "measured"
    except Exception:
        bf16, hbm, src = 1590.0, 6650.0, "fallback"
    try:
        i8 = json.load(open(os.path.join(ROOT, "profiles", "int8_peak.json")))["int8_tops_burst"]
    except Exception:
        i8 = 2 * bf16
    return bf16, hbm, i8, src


def graph_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    torch.cuda.set_device(0)
    bf16, hbm, i8, src = peaks()
    digit = i8 / 10
    dims = [int(a) for a in sys.argv[1:]] or [256, 512, 768, 1024, 2048, 3072, 4096, 8192]
    rows = []
    for d in dims:
        g = torch.Generator(device="cuda").manual_seed(d)
        x = torch.randn((d, N), generator=g, device="cuda").to(torch.bfloat16)
        f = torch.empty((d, d), device="cuda")
        t_syrk = graph_ms(lambda: K.syrk([(x, f, 1.0 / N, False)], fill_upper=False))
        # a grouped launch of 8 factors of this size (how K-FAC work items call it)
        xs8 = [x] * 8
        fs8 = [torch.empty((d, d), device="cuda") for _ in range(8)] if d <= 4096 else [f]
        t_syrk8 = graph_ms(lambda: K.syrk([(xi, fi, 1.0 / N, False) for xi, fi in zip(xs8, fs8)], fill_upper=False))
        n8 = len(fs8)
        fl_syrk = d * (d + 1) * N
        by_syrk = 2 * d * N + 2 * d * (d + 1)
        K.syrk([(x, f, 1.0 / N, False)], fill_upper=True)
        nb = 8 if d <= 4096 else 2
        mats = [f] * nb
        outs = [torch.empty_like(f) for _ in range(nb)]
        digs = [torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda") for _ in range(nb)]
        t_inv1 = graph_ms(lambda: K.damped_inverse_batched(mats[:1], 0.1, outs[:1], digs[:1], check=False), reps=3)
        t_invb = graph_ms(lambda: K.damped_inverse_batched(mats, 0.1, outs, digs, check=False), reps=3)
        a = K.SlicedMatrix(outs[0], digs[0])
        grad = torch.randn((d, d), generator=g, device="cuda")
        w = torch.zeros((d, d), device="cuda")
        t_prec = graph_ms(lambda: K.precondition_update_sliced([(w, grad, a, a, 1e-3)]))
        fl_prec = 4 * d ** 3
        r = {"d": d, "n": N,
             "syrk_ms": t_syrk, "syrk_tflops": fl_syrk / t_syrk / 1e9, "syrk_gbs": by_syrk / t_syrk / 1e6,
             "syrk_bound": "hbm" if fl_syrk / by_syrk < bf16 * 1e3 / hbm else "tensor",
             "syrk_grouped": n8, "syrk_grouped_ms": t_syrk8, "syrk_grouped_tflops": n8 * fl_syrk / t_syrk8 / 1e9,
             "inverse_1_ms": t_inv1, "inverse_1_tflops": d ** 3 / t_inv1 / 1e9,
             "inverse_b_ms": t_invb, "inverse_batch_tflops": nb * d ** 3 / t_invb / 1e9, "inverse_batch": nb,
             "prec_ms": t_prec, "prec_tflops": fl_prec / t_prec / 1e9}
        r["syrk_frac"] = (r["syrk_gbs"] / hbm) if r["syrk_bound"] == "hbm" else (r["syrk_tflops"] / bf16)
        r["syrk_grouped_frac"] = r["syrk_grouped_tflops"] / bf16
        r["inverse_batch_frac_digit"] = r["inverse_batch_tflops"] / digit
        r["prec_frac_digit"] = r["prec_tflops"] / digit
        rows.append(r)
        print(json.dumps(r), flush=True)
        del x, f, outs, digs, grad, w, mats, fs8
        torch.cuda.empty_cache()
    print(f"\npeaks ({src}, burst): bf16 dense {bf16} TFLOP/s, HBM {hbm} GB/s, int8 dense {i8} TOP/s -> "
          f"int8-digit fp32-accurate ceiling {digit:.0f} TFLOP/s\n")
    print("| d | SYRK ms | SYRK TFLOP/s | SYRK GB/s | bound | frac | SYRK x8 grouped TFLOP/s | frac | inverse x1 ms | "
          "x1 TFLOP/s | inverse xB ms | xB TFLOP/s | xB frac(digit) | precond ms | precond TFLOP/s | frac(digit) |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['d']} | {r['syrk_ms']:.3f} | {r['syrk_tflops']:.0f} | {r['syrk_gbs']:.0f} | {r['syrk_bound']} | "
              f"{r['syrk_frac']:.2f} | {r['syrk_grouped_tflops']:.0f} | {r['syrk_grouped_frac']:.2f} | "
              f"{r['inverse_1_ms']:.2f} | {r['inverse_1_tflops']:.1f} | "
              f"{r['inverse_b_ms']:.2f} x{r['inverse_batch']} | "
              f"{r['inverse_batch_tflops']:.1f} | {r['inverse_batch_frac_digit']:.2f} | {r['prec_ms']:.3f} | "
              f"{r['prec_tflops']:.0f} | {r['prec_frac_digit']:.2f} |")


if __name__ == "__main__":
    main()
