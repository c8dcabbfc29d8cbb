"""Dump pf_slice outputs for a fixed set of inputs (bit-exact A/B of slicing
implementations: run once per library via PF_LIB_PATH, compare the npz)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2211_14133_b200 import _lib as L, kfac as K
torch.cuda.set_device(0)
out = {}
g = torch.Generator(device="cuda").manual_seed(5)
for (rows, k, kind) in [(64, 100, "n"), (300, 1024, "n"), (257, 1500, "mix"), (128, 4096, "n"), (64, 8192, "mix"),
                        (33, 2048, "ties"), (16, 4096, "tiny")]:
    x = torch.randn(rows, k, generator=g, device="cuda")
    if kind == "mix":
        x = x * torch.exp(torch.randn(rows, 1, generator=g, device="cuda") * 20)
        x[::7] = 0
        x[3, ::3] = -x[3, ::3]
    if kind == "ties":
        m = x.abs().amax(1, keepdim=True)
        e = torch.frexp(m)[1].float()
        q = torch.round(x * torch.exp2(28 - e)) + 0.5
        x = q * torch.exp2(e - 28)
    if kind == "tiny":
        x = x * 1e-38
    buf = torch.zeros(K.slice_bytes(rows, k), dtype=torch.uint8, device="cuda")
    L.check(L.lib().pf_slice(x.data_ptr(), rows, k, k, buf.data_ptr(), K._stream()), "slice")
    torch.cuda.synchronize()
    out[f"{rows}x{k}{kind}"] = buf.cpu().numpy()
np.savez(sys.argv[1], **out)
print("dumped", len(out))
