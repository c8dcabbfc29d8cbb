"""Diagnostic: per-tile error of the LAUUM (X^T X) step of the damped inverse."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2211_14133_b200 import kfac as K
from oracle import ref as R

d = 1024
x = torch.from_numpy(R.orc_symmetric(1300, (d, 4096), 3 ** 0.5)).to(torch.bfloat16).double()
m = (x @ x.T / 4096).float().cuda()
inv = K.cholesky_spd_inverse(m, 0.1).double()
ws = K._WS._bufs[(0, "inverse")]
ld = d
plane = ((ld * d * 4) + 255) // 256 * 256
X = ws[2 * plane: 2 * plane + ld * d * 4].view(torch.float32).view(d, ld).double()
XT = ws[3 * plane: 3 * plane + ld * d * 4].view(torch.float32).view(d, ld).double()
Xl = torch.tril(X)
ref = Xl.T @ Xl
E = (inv - ref).abs()
print("max err", E.max().item(), "max |ref|", ref.abs().max().item())
T = d // 128
for tm in range(T):
    print(" ".join(f"{E[tm*128:(tm+1)*128, tn*128:(tn+1)*128].max().item():.1e}" for tn in range(T)))
# XT consistency with X
print("XT upper vs X^T:", (torch.triu(XT) - Xl.T).abs().max().item())
# our GEMM on a plain product through precondition: P = B G A with B = X^T-like
g = torch.triu(XT).float().contiguous()
p = K.precondition(g, torch.eye(d, device='cuda'), torch.eye(d, device='cuda')).double()
print("identity-precondition roundtrip err:", (p - g.double()).abs().max().item())
sl = K.slice_matrix(torch.triu(XT).float().contiguous())
print("sliced exps first rows:", sl.digits[4 * d * d: 4 * d * d + 64].view(torch.int32)[:16].tolist())
