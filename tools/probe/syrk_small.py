import sys, torch
sys.path.insert(0, ".")
from paper_2211_14133_b200 import kfac as K
torch.cuda.set_device(0)
for d, n in ((128, 64), (128, 4096), (1024, 4096), (2048, 4096), (4096, 4096)):
    x = torch.randn((d, n), device="cuda").to(torch.bfloat16)
    f = torch.empty((d, d), device="cuda")
    for _ in range(3):
        K.syrk([(x, f, 1.0, False)], fill_upper=False)
    torch.cuda.synchronize()
print("ok")
