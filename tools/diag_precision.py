"""Where does the damped inverse lose accuracy?  (development diagnostic)

    python tools/diag_precision.py [d]

Runs one pf_damped_inverse on a bench-like factor (unit-variance bf16 tapes,
n = 4096, lambda = 0.1), reads the intermediate planes back out of the
workspace (damped/updated A, strictly-lower L, X = L^-1) and reports in fp64:
  * the final residual max|(M + lambda I) Minv - I|;
  * the residual of X^T X formed exactly from the GPU's X (LAUUM excluded);
  * the leaf error max|X_kk A_kk X_kk^T - I| per 128-block against an fp32
    cuSOLVER Cholesky + inverse of the SAME block;
  * the Cholesky backward error max|L L^T - M| (L_kk = X_kk^-1);
  * the same algorithm emulated with fp64 products rounded to fp32 once.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2211_14133_b200 import kfac as K  # noqa: E402

LAM = 0.1
B = 128


def a256(x):
    return (x + 255) // 256 * 256


def main():
    d = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    torch.cuda.set_device(0)
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.randn((d, 4096), generator=g, device="cuda").to(torch.bfloat16).float()
    m = (x @ x.T) / 4096
    out = K.damped_inverse_batched([m], LAM)[0]
    torch.cuda.synchronize()
    ws = K._WS._bufs[(0, "inverse")]
    ld = (d + 3) // 4 * 4
    plane = a256(ld * d * 4)
    f = ws.view(torch.float32)

    def pl(i):
        return f[i * plane // 4: i * plane // 4 + d * ld].view(d, ld)[:, :d].double()

    Aw, Lw, Xw = pl(0), pl(1), pl(2)
    I = torch.eye(d, device="cuda", dtype=torch.float64)
    M = torch.tril(m.double()) + torch.tril(m.double(), -1).T + LAM * I
    print(f"d = {d}")
    print(f"final residual              {(M @ out.double() - I).abs().max().item():.3e}")
    X = torch.tril(Xw)
    print(f"residual of X^T X (exact)   {(M @ (X.T @ X) - I).abs().max().item():.3e}")
    print(f"max|X M X^T - I|            {(X @ M @ X.T - I).abs().max().item():.3e}")
    Lf = torch.zeros_like(M)
    worst_leaf, worst_ref = 0.0, 0.0
    for k in range(0, d, B):
        n = min(B, d - k)
        akk = torch.tril(Aw[k:k + n, k:k + n])
        akk = akk + torch.tril(akk, -1).T
        xkk = X[k:k + n, k:k + n]
        e = (xkk @ akk @ xkk.T - torch.eye(n, device="cuda", dtype=torch.float64)).abs().max().item()
        lc = torch.linalg.cholesky(akk.float())
        xc = torch.linalg.inv(lc).double()
        er = (xc @ akk @ xc.T - torch.eye(n, device="cuda", dtype=torch.float64)).abs().max().item()
        worst_leaf, worst_ref = max(worst_leaf, e), max(worst_ref, er)
        Lf[k:k + n, k:k + n] = torch.linalg.inv(xkk)
        if k + n < d:
            Lf[k + n:, k:k + n] = Lw[k + n:, k:k + n]
    print(f"leaf max|X A X^T - I|       {worst_leaf:.3e}   (fp32 cuSOLVER on the same blocks: {worst_ref:.3e})")
    print(f"chol backward max|LL^T-M|   {(Lf @ Lf.T - M).abs().max().item():.3e}")
    # emulation: fp64 products rounded to fp32 once, fp32 cuSOLVER leaves
    f32 = lambda t: t.float().double()  # noqa: E731
    Ae = f32(M.clone())
    Le = torch.zeros_like(M)
    Xe = torch.zeros_like(M)
    for k in range(0, d, B):
        n = min(B, d - k)
        akk = torch.tril(Ae[k:k + n, k:k + n])
        akk = akk + torch.tril(akk, -1).T
        lkk = torch.linalg.cholesky(akk.float())
        xkk = torch.linalg.inv(lkk)
        xkk = torch.tril(xkk).double()
        Le[k:k + n, k:k + n] = lkk.double()
        Xe[k:k + n, k:k + n] = xkk
        if k + n < d:
            l21 = f32(Ae[k + n:, k:k + n] @ xkk.T)
            Le[k + n:, k:k + n] = l21
            Ae[k + n:, k + n:] = f32(Ae[k + n:, k + n:] - l21 @ l21.T)

    def trtri(o, nn):
        if nn <= B:
            return
        n1 = B * ((nn + 2 * B - 1) // (2 * B))
        trtri(o, n1)
        trtri(o + n1, nn - n1)
        T = f32(Le[o + n1:o + nn, o:o + n1] @ Xe[o:o + n1, o:o + n1])
        Xe[o + n1:o + nn, o:o + n1] = f32(-(Xe[o + n1:o + nn, o + n1:o + nn] @ T))

    trtri(0, d)
    Me = f32(Xe.T @ Xe)
    print(f"emulated final residual     {(M @ Me - I).abs().max().item():.3e}")
    print(f"emulated X^T X (exact)      {(M @ (Xe.T @ Xe) - I).abs().max().item():.3e}")
    print(f"emulated chol backward      {(Le @ Le.T - M).abs().max().item():.3e}")
    print(f"max|X - X_emul| / max|X|    {(X - Xe).abs().max().item() / Xe.abs().max().item():.3e}")


if __name__ == "__main__":
    main()
