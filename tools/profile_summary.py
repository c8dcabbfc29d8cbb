"""Summarise ncu --set full reports (key metrics per kernel) into markdown.

    python tools/profile_summary.py OUT.md rep1.ncu-rep [rep2 ...]
"""
import csv
import io
import subprocess
import sys

WANT = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
    ("sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "tensor hmma cycles (TPC avg)"),
    ("sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "tensor imma cycles (TPC avg)"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("smsp__inst_executed.sum", "instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
]


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u = r[0], r[1]
    for row in r[2:]:
        d = {}
        for k, un, v in zip(h, u, row):
            d[k] = (v, un)
        yield d


def main():
    out, reps = sys.argv[1], sys.argv[2:]
    lines = []
    for rep in reps:
        for d in rows(rep):
            name = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"### `{name[:120]}`  ({rep.split('/')[-1]})\n")
            lines.append("| metric | value | unit |\n|---|---|---|")
            for key, label in WANT:
                for k, (v, un) in d.items():
                    if k.endswith(key):
                        lines.append(f"| {label} (`{key}`) | {v} | {un} |")
                        break
            lines.append("")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
