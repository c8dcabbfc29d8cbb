import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2211_14133_b200 import kfac as K
from oracle import ref as R
torch.backends.cuda.matmul.allow_tf32 = False
for d in (32, 64, 100, 128, 256, 512, 1024):
    x = torch.from_numpy(R.orc_symmetric(300+d, (d, 2*d), 3**0.5)).to(torch.bfloat16).double()
    m = (x @ x.T / (2*d)).float().cuda()
    inv = K.cholesky_spd_inverse(m, 0.1).double()
    a = m.double() + 0.1*torch.eye(d, device='cuda', dtype=torch.float64)
    r = (a @ inv - torch.eye(d, device='cuda', dtype=torch.float64)).abs().max().item()
    ref = torch.linalg.inv(a)
    rel = (torch.linalg.norm(inv-ref)/torch.linalg.norm(ref)).item()
    # fp32 torch (cuSOLVER) for comparison
    i32 = torch.cholesky_inverse(torch.linalg.cholesky(a.float())).double()
    r32 = (a @ i32 - torch.eye(d, device='cuda', dtype=torch.float64)).abs().max().item()
    print(f"d={d} residual={r:.2e} rel={rel:.2e}  cusolver-fp32 residual={r32:.2e}")
# GEMM accuracy of the 3xTF32 path vs K via precondition with A^-1 = I
for k in (64, 256, 1024, 4096):
    g = torch.randn(256, k, device='cuda'); b = torch.randn(256, 256, device='cuda')
    p = K.precondition(g, torch.eye(k, device="cuda"), b).double()
    ref = b.double() @ g.double()
    print("K", k, "rel", (torch.linalg.norm(p-ref)/torch.linalg.norm(ref)).item())
