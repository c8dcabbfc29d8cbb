"""Top source lines by warp-stall samples from an ncu report (needs -lineinfo):
    python tools/ncu_lines.py report.ncu-rep [N]"""
import csv, io, subprocess, sys

def main():
    rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None; res = []; fname = ""
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path": fname = r[1].split("/")[-1]
        if len(r) > 5 and r[0] == "Line No": hdr = r; continue
        if hdr and len(r) == len(hdr) and r[0] not in ("", "Line No"):
            d = dict(zip(hdr, r))
            try: s = int(d["Warp Stall Sampling (All Samples)"]); ie = int(d["Instructions Executed"])
            except ValueError: continue
            res.append((s, ie, fname, r[0], r[1][:90]))
    tot = sum(x[0] for x in res) or 1
    print(f"total samples {tot}")
    for s, ie, f, ln, src in sorted(res, reverse=True)[:n]:
        print(f"{100*s/tot:5.1f}% {ie:8d} {f}:{ln:5s} {src}")

if __name__ == "__main__":
    main()
