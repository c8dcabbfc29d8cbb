import torch, time
torch.cuda.set_device(0)
n = 201 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
hb = torch.empty(50 * 1024 * 1024, dtype=torch.uint8).pin_memory()
db = torch.empty(50 * 1024 * 1024, dtype=torch.uint8, device="cuda")
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def one(): d.copy_(h, non_blocking=True)
def two():
    half = n // 2
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
def with_d2h():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s3): hb.copy_(db, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s3)
for name, fn in [("one", one), ("two streams", two), ("h2d+d2h", with_d2h)]:
    ms = t(fn); print(f"{name:12s} {ms:.3f} ms  {n / ms / 1e6:.1f} GB/s")

# the same copies while the SMs run the K-FAC step's kind of load (big GEMMs)
a = torch.randn(8192, 8192, device="cuda")
comp = torch.cuda.Stream()
def busy():
    with torch.cuda.stream(comp):
        for _ in range(6):
            a @ a
def one_busy():
    busy()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
        hb.copy_(db, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(comp)
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
with torch.cuda.stream(s1):
    e0.record(s1); d.copy_(h, non_blocking=True); e1.record(s1)
busy()
torch.cuda.synchronize()
print(f"h2d under compute: {e0.elapsed_time(e1):.3f} ms  {n / e0.elapsed_time(e1) / 1e6:.1f} GB/s")
