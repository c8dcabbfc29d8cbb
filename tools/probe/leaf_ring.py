"""In-situ leaf timing inside one damped-inverse call (CUDA graph replay):
library built with -DPF_LEAF_RING into tools/probe/leafring/ by
    make -C paper_2211_14133_b200 OUT=$PWD/tools/probe/leafring OBJ=/tmp/leafring NVFLAGS_EXTRA=-DPF_LEAF_RING
Prints per leaf launch (CTA 0): wait after entry, load, compute+store, in ns,
the clock64 cycles entry->end, and the implied SM clock."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ.setdefault("PF_LIB_PATH", os.path.join(ROOT, "tools/probe/leafring/libpf_b200.so"))
import torch
from paper_2211_14133_b200 import kfac as K, _lib as L
torch.cuda.set_device(0)
lib = L.lib()
lib.pf_leaf_ring_read.restype = C.c_int
spec = [tuple(int(v) for v in p.split(":")) for p in (sys.argv[1] if len(sys.argv) > 1 else "4096:1").split(",")]
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
h = (C.c_longlong * 512)()
lib.pf_leaf_ring_read(h)
g.replay()
torch.cuda.synchronize()
n = min(64, lib.pf_leaf_ring_read(h))
recs = sorted((tuple(h[8 * i: 8 * i + 8]) for i in range(n)), key=lambda r: r[0])
t00 = recs[0][0]
tot = [0, 0, 0]
for r in recs:
    wait, load, rest, store = r[1] - r[0], r[2] - r[1], r[6] - r[2], r[3] - r[6]
    cyc = r[5] - r[4]
    mhz = cyc / max(1, r[3] - r[0]) * 1e3
    tot[0] += wait; tot[1] += load; tot[2] += rest
    print(f"col0 {r[7]:5d} @ {(r[0] - t00) / 1e3:8.1f} us  wait {wait / 1e3:6.1f}  load {load / 1e3:5.1f}  "
          f"compute {rest / 1e3:5.1f}  store {store / 1e3:5.1f} us  cycles {cyc:6d}  ~{mhz:5.0f} MHz")
print(f"{n} leaves: mean wait {tot[0] / n / 1e3:.1f} load {tot[1] / n / 1e3:.1f} compute+store {tot[2] / n / 1e3:.1f} us (compute/store split per line)")
