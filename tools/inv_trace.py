"""Timeline of one persistent inversion launch (PF_INV_TRACE):
    python tools/inv_trace.py d:count[,d:count...]
Prints per-phase span (first ready -> last done) and gaps, plus per-type totals."""
import csv, os, sys, collections
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = "/tmp/inv_trace.csv"
os.environ["PF_INV_TRACE"] = path
import torch
from paper_2211_14133_b200 import kfac as K
torch.cuda.set_device(0)
K.L.check(K.L.lib().pf_set_inverse_mode(1), "mode")  # the trace comes from the persistent executor
spec = [tuple(int(v) for v in p.split(":")) for p in (sys.argv[1] if len(sys.argv) > 1 else "256:2").split(",")]
mats = []
for d, c in spec:
    for j in range(c):
        x = torch.randn(d, 4096, device="cuda").to(torch.bfloat16).float()
        mats.append(x @ x.T / 4096)
for _ in range(3):
    K.damped_inverse_batched(mats, 0.1, check=False)
torch.cuda.synchronize()
rows = list(csv.DictReader(open(path)))
t0 = min(int(r["claimed_ns"]) for r in rows)
names = {0: "damp", 1: "slice", 2: "leaf", 3: "gemm"}
ph = collections.OrderedDict()
for r in rows:
    p = int(r["phase"])
    e = ph.setdefault(p, dict(type=names[int(r["type"])], n=0, ready=1e30, claim=1e30, done=0, work=0))
    e["n"] += 1
    e["ready"] = min(e["ready"], int(r["ready_ns"]) - t0)
    e["claim"] = min(e["claim"], int(r["claimed_ns"]) - t0)
    e["done"] = max(e["done"], int(r["done_ns"]) - t0)
    e["work"] = max(e["work"], int(r["done_ns"]) - int(r["ready_ns"]))
prev = 0
tot = collections.Counter()
limit = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for i, (p, e) in enumerate(ph.items()):
    if i < limit:
        print(f"phase {p:4d} {e['type']:5s} x{e['n']:4d}  ready {e['ready']/1e3:8.1f}  done {e['done']/1e3:8.1f} us"
              f"  span {(e['done']-e['ready'])/1e3:6.1f}  max task {e['work']/1e3:6.1f}  gap-from-prev {(e['ready']-prev)/1e3:6.1f}")
    prev = e["done"]
    tot[e["type"]] += e["done"] - e["ready"]
end = max(e["done"] for e in ph.values())
lv = [r for r in rows if r["type"] == "2"]
for r in lv[:4]:
    ns = int(r["done_ns"]) - int(r["ready_ns"]); cyc = int(r["mma_issued"] or 0)
    print(f"leaf task {r['task']}: {ns/1e3:.1f} us, {cyc} cycles -> {cyc/ns:.2f} GHz effective")
g = [r for r in rows if r["type"] == "3"]
if g:
    print("GEMM tile sub-phases (us, from ready): acc_ready / pre_wait / staged / epi_end / done")
    for r in g[:12]:
        rd = int(r["ready_ns"])
        f = lambda k: (int(r[k]) - rd) / 1e3 if int(r[k]) else float("nan")
        print(f"  phase {r['phase']:>4} tile {r['b']:>4}: {f('mma_issued'):6.1f} {f('pre_wait'):6.1f} {f('acc_ready'):6.1f} {f('epi_end'):6.1f} {f('done_ns'):6.1f}")
print("total", end / 1e3, "us;", {k: round(v / 1e3, 1) for k, v in tot.items()})
