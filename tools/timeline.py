"""CUPTI kernel timeline (torch.profiler) of one damped-inverse call, replayed
from a CUDA graph exactly as bench.py runs it:

    python tools/timeline.py [d:count,...]   (default 4096:2,1024:10)

Prints the span, the busy time (union of kernel intervals), per-kernel-name
totals, and the gaps between consecutive kernels on the critical chain.
Development tool; numbers under a profiler are not bench values.
"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402


def main():
    torch.cuda.set_device(0)
    spec = [tuple(int(v) for v in p.split(":")) for p in (sys.argv[1] if len(sys.argv) > 1 else "4096:2,1024:10").split(",")]
    mats, outs, digs = [], [], []
    for d, c in spec:
        for _ in range(c):
            x = torch.randn(d, 4096, device="cuda").to(torch.bfloat16).float()
            mats.append(x @ x.T / 4096)
            outs.append(torch.empty(d, d, device="cuda"))
            digs.append(torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda"))
    call = lambda: K.damped_inverse_batched(mats, 0.1, outs, digs, check=False)  # noqa: E731
    call()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        call()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type.name == "CUDA" and e.time_range.elapsed_us() > 0]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    t1 = max(e.time_range.end for e in ev)
    # union of busy intervals
    busy, cur_s, cur_e = 0.0, None, None
    for e in ev:
        a, b = e.time_range.start, e.time_range.end
        if cur_s is None or a > cur_e:
            if cur_s is not None:
                busy += cur_e - cur_s
            cur_s, cur_e = a, b
        else:
            cur_e = max(cur_e, b)
    busy += cur_e - cur_s
    print(f"span {t1 - t0:.1f} us, busy (union) {busy:.1f} us, kernels {len(ev)}")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for e in ev:
        k = e.name.split("(")[0].replace("void ", "")[:40]
        agg[k][0] += 1
        agg[k][1] += e.time_range.elapsed_us()
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:40s} {n:5d} launches {t:9.1f} us (sum)")
    # idle gaps (no kernel running at all)
    gaps = []
    cur_e = ev[0].time_range.end
    for e in ev[1:]:
        if e.time_range.start > cur_e:
            gaps.append(e.time_range.start - cur_e)
        cur_e = max(cur_e, e.time_range.end)
    if gaps:
        gaps.sort()
        print(f"idle gaps: {len(gaps)} totalling {sum(gaps):.1f} us; median {gaps[len(gaps) // 2]:.2f} us, max {gaps[-1]:.1f} us")
    # concurrency profile: time with exactly one kernel running
    pts = sorted([(e.time_range.start, 1) for e in ev] + [(e.time_range.end, -1) for e in ev])
    level, last, single = 0, t0, 0.0
    for t, dlt in pts:
        if level == 1:
            single += t - last
        level += dlt
        last = t
    print(f"time with exactly one kernel running: {single:.1f} us ({100 * single / (t1 - t0):.0f}% of span)")
    # marginal (critical-path) attribution: kernels sorted by end time, each
    # charged end_k - end_{k-1}; with PDL a kernel starts early, so its own
    # duration overstates its cost
    by_end = sorted(ev, key=lambda e: e.time_range.end)
    marg = collections.defaultdict(lambda: [0, 0.0])
    prev = t0
    for e in by_end:
        k = e.name.split("(")[0].replace("void ", "")[:40]
        grid = ""
        marg[k][0] += 1
        marg[k][1] += e.time_range.end - prev
        prev = e.time_range.end
    if os.environ.get("PF_TL_DUMP"):
        lo, hi = (int(v) for v in os.environ["PF_TL_DUMP"].split(":"))
        for e in by_end[lo:hi]:
            print(f"  {e.name.split('(')[0][:36]:36s} s{getattr(e, 'device_resource_id', -1):<4} start {e.time_range.start - t0:9.1f} end {e.time_range.end - t0:9.1f} dur {e.time_range.elapsed_us():7.1f}")
    print("marginal time by kernel (sum of end-to-end deltas):")
    for k, (n, t) in sorted(marg.items(), key=lambda x: -x[1][1]):
        print(f"  {k:40s} {n:5d} {t:9.1f} us  ({t / n:6.2f} us each)")


if __name__ == "__main__":
    main()
