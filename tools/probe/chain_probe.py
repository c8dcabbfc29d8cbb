"""globaltimer probe of the chain steps (chain.cuh) inside one damped inverse;
library built with -DPF_CHAIN_PROBE into tools/probe/chainprobe/ by
tools/probe/build_chainprobe.sh.  Prints, per launch (CTA 0 of the first
cluster): entry -> griddepcontrol.wait done -> operands staged -> step 1 ->
gather -> step 2 -> leaf done, in ns, and the gap since the previous step."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["PF_LIB_PATH"] = os.path.join(ROOT, "tools/probe/chainprobe/libpf_b200.so")
import torch
from paper_2211_14133_b200 import kfac as K, _lib as L
torch.cuda.set_device(0)
lib = L.lib()
lib.pf_chain_probe_read.restype = C.c_int
spec = [tuple(int(v) for v in p.split(":")) for p in (sys.argv[1] if len(sys.argv) > 1 else "4096:1").split(",")]
mats, outs, digs = [], [], []
for d, cnt in spec:
    for i in range(cnt):
        x = torch.randn(d, 4096, device="cuda").to(torch.bfloat16).float()
        mats.append(x @ x.T / 4096)
        outs.append(torch.empty(d, d, device="cuda"))
        digs.append(torch.empty(K.slice_bytes(d, d), dtype=torch.uint8, device="cuda"))
call = lambda: K.damped_inverse_batched(mats, 0.1, outs, digs, check=False)  # noqa: E731
for _ in range(3):
    call()
torch.cuda.synchronize()
h = (C.c_longlong * 512)()
lib.pf_chain_probe_read(h)
call()
torch.cuda.synchronize()
n = min(64, lib.pf_chain_probe_read(h))
names = ["wait", "staged", "step1", "gather", "step2", "leaf"]
prev = None
for i in range(n):
    r = h[8 * i: 8 * i + 8]
    rel = [r[j] - r[j - 1] for j in range(1, 7)]
    gap = (r[0] - prev) if prev else 0
    prev = r[6]
    print(f"{i:2d} " + " ".join(f"{nm} {v / 1000:6.2f}" for nm, v in zip(names, rel)) + f"  total {(r[6] - r[0]) / 1000:6.2f} us  (entry - prev end {gap / 1000:6.2f} us)")
