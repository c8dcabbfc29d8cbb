"""Clock-stamp probe of one small digit GEMM (library built with -DPF_GEMM_PROBE)."""
import ctypes as C, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
os.environ["PF_LIB_PATH"] = os.path.join(ROOT, "tools/probe/gemmprobe/libpf_b200.so")
import torch
from paper_2211_14133_b200 import kfac as K, _lib as L
torch.cuda.set_device(0)
lib = L.lib()
for d in (128, 512, 2048):
    a = torch.eye(d, device="cuda"); g = torch.randn(d, d, device="cuda"); out = torch.empty_like(g)
    nb = K.precondition_workspace_bytes(d, d); ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        lib.pf_precondition(a.data_ptr(), g.data_ptr(), a.data_ptr(), out.data_ptr(), d, d, ws.data_ptr(), nb, K._stream())
    torch.cuda.synchronize()
    h = (C.c_longlong * 16)()
    lib.pf_gemm_probe_read(h)
    names = ["entry", "prologue", "first data", "mma issued", "acc ready", "epilogue end", "dealloc"]
    print(f"d={d} (last GEMM of precondition, CTA 0):", " ".join(f"{names[i]}+{h[i]-h[0]}" for i in range(1, 7)))
