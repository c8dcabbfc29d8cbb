"""Dump damped-inverse outputs (and digit forms) for fixed inputs: bit-exact
A/B of two builds via PF_LIB_PATH."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2211_14133_b200 import kfac as K
torch.cuda.set_device(0)
g = torch.Generator(device="cuda").manual_seed(3)
mats = []
for d in (300, 1024, 1024, 2048):
    x = torch.randn(d, 2048, generator=g, device="cuda")
    mats.append(x @ x.T / 2048)
outs = [torch.empty_like(m) for m in mats]
digs = [torch.empty(K.slice_bytes(m.shape[0], m.shape[0]), dtype=torch.uint8, device="cuda") for m in mats]
K.damped_inverse_batched(mats, 0.1, outs, digs, check=True)
w = torch.randn(1024, 2048, generator=g, device="cuda")
gr = torch.randn(1024, 2048, generator=g, device="cuda")
torch.cuda.synchronize()
np.savez(sys.argv[1], **{f"inv{i}": o.cpu().numpy() for i, o in enumerate(outs)},
         **{f"dig{i}": d.cpu().numpy() for i, d in enumerate(digs)})
print("ok")
