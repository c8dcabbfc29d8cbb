"""Top source lines (CUDA view) of an ncu report by warp-stall samples:
    python tools/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=" + (sys.argv[3] if len(sys.argv) > 3 else "sass")],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
blocks, cur = [], []
for ln in lines:
    if ln.startswith('"File Name"') or ln.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [ln]
    else:
        cur.append(ln)
if cur:
    blocks.append(cur)
rows = []
for b in blocks:
    fname = b[0]
    r = list(csv.reader(io.StringIO("\n".join(b[1:]))))
    if not r or "Source" not in r[0]:
        continue
    h = r[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    li = h.index("Line No") if "Line No" in h else h.index("Address")
    stall_cols = [i for i, k in enumerate(h) if k.startswith("stall_")]
    for row in r[1:]:
        try:
            s = float(row[si] or 0)
        except (ValueError, IndexError):
            continue
        if s > 0:
            top = sorted(((float(row[i] or 0), h[i]) for i in stall_cols), reverse=True)[:3]
            rows.append((s, fname.split(",")[-1].strip('"').split("/")[-1], row[li], row[h.index("Source")].strip()[:90],
                         " ".join(f"{k[6:]}={v:.0f}" for v, k in top if v > 0)))
tot = sum(x[0] for x in rows)
for s, f, l, src, st in sorted(rows, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}% {f}:{l:>4s} {src:90s} {st}")
