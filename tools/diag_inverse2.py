"""Diagnostic: where does the damped-inverse error come from?  Reads the
workspace intermediates (X = L^-1) after one call and compares per 128-block
row against an fp64 Cholesky."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_2211_14133_b200 import kfac as K
from oracle import ref as R

for d in (256, 1024):
    x = torch.from_numpy(R.orc_symmetric(300 + d, (d, 4096), 3 ** 0.5)).to(torch.bfloat16).double()
    m = (x @ x.T / 4096).float().cuda()
    inv = K.cholesky_spd_inverse(m, 0.1).double()
    a = m.double() + 0.1 * torch.eye(d, device='cuda', dtype=torch.float64)
    L = torch.linalg.cholesky(a)
    Xref = torch.linalg.inv(L)
    ws = K._WS._bufs[(0, "inverse")]
    ld = (d + 3) // 4 * 4
    plane = ((ld * d * 4) + 255) // 256 * 256
    X = ws[2 * plane: 2 * plane + ld * d * 4].view(torch.float32).view(d, ld)[:, :d].double()
    XT = ws[3 * plane: 3 * plane + ld * d * 4].view(torch.float32).view(d, ld)[:, :d].double()
    err = (torch.tril(X) - Xref).abs()
    print(f"d={d}: max|X-Xref| {err.max():.2e}  max|XT^T - Xref| {(torch.triu(XT).T - Xref).abs().max():.2e}")
    for b in range(0, d, 128):
        blk = err[b:b + 128, :b + 128]
        diag = err[b:b + 128, b:b + 128].max().item()
        print(f"  rows {b:5d}: max err {blk.max().item():.2e}  diag-block {diag:.2e}")
    # residual using exact X
    Xr = torch.tril(X)
    minv = Xr.T @ Xr
    print("  residual with fp64 LAUUM of our X:", (a @ minv - torch.eye(d, device='cuda', dtype=torch.float64)).abs().max().item())
    print("  residual of our inverse:", (a @ inv - torch.eye(d, device='cuda', dtype=torch.float64)).abs().max().item())
    # fp32-rounded exact inverse
    ex = torch.linalg.inv(a).float().double()
    print("  residual of fp32-rounded exact inverse:", (a @ ex - torch.eye(d, device='cuda', dtype=torch.float64)).abs().max().item())
