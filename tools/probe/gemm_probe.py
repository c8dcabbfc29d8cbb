"""globaltimer probe of the small beta != 0 digit GEMMs (the per-panel diagonal
updates) inside one 2x4096 damped inverse; library built with -DPF_GEMM_PROBE
into tools/probe/gemmprobe/.  Prints, per launch (CTA 0): entry -> after
griddepcontrol.wait -> first TMA data -> MMAs issued -> accumulator ready ->
epilogue end, in ns."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["PF_LIB_PATH"] = os.path.join(ROOT, "tools/probe/gemmprobe/libpf_b200.so")
import torch
from paper_2211_14133_b200 import kfac as K, _lib as L
torch.cuda.set_device(0)
lib = L.lib()
lib.pf_gemm_probe_read.restype = C.c_int
d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mats, outs, digs = [], [], []
for i in range(cnt):
    x = torch.randn(d, 4096, device="cuda").to(torch.bfloat16).float()
    mats.append(x @ x.T / 4096)
    outs.append(torch.empty(d, d, device="cuda"))
    digs.append(torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda"))
call = lambda: K.damped_inverse_batched(mats, 0.1, outs, digs, check=False)  # noqa: E731
for _ in range(3):
    call()
torch.cuda.synchronize()
h = (C.c_longlong * 1024)()
lib.pf_gemm_probe_read(h)
call()
torch.cuda.synchronize()
n = min(64, lib.pf_gemm_probe_read(h))
names = ["wait-done", "first-data", "mma-issued", "acc-ready", "epi-end"]
prev = None
for i in range(n):
    r = h[16 * i: 16 * i + 16]
    rel = [r[j] - r[0] for j in range(1, 6)]
    epi = [r[j] - r[4] for j in range(6, 14)]
    gap = (r[1] - prev) if prev else 0
    prev = r[5]
    print(f"{i:2d} {r[14]}x{r[15]} " + " ".join(f"{nm}+{v}" for nm, v in zip(names, rel)) + f"  (since prev end {gap} ns)"
          + "  epi: scales+%d tmem0+%d chunks %s tmem1 %d..%d" % (epi[0], epi[1], [e for e in epi[2:6]], epi[6], epi[7]))
