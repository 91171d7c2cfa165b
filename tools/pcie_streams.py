import time, torch
MB = 1 << 20
hs = [torch.empty(360 * MB // 8, dtype=torch.float64).pin_memory() for _ in range(2)]
ds = [torch.empty_like(h, device="cuda") for h in hs]
ss = [torch.cuda.Stream() for _ in range(4)]
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
def one():
    for h, d in zip(hs, ds): d.copy_(h, non_blocking=True)
def two():
    for i, (h, d) in enumerate(zip(hs, ds)):
        with torch.cuda.stream(ss[i]): d.copy_(h, non_blocking=True)
def four():
    for i in range(4):
        h, d = hs[i % 2], ds[i % 2]
        n = h.numel() // 2; sl = slice((i // 2) * n, (i // 2 + 1) * n)
        with torch.cuda.stream(ss[i]): d[sl].copy_(h[sl], non_blocking=True)
for name, f in (("1 stream", one), ("2 streams", two), ("4 streams", four)):
    t = timed(f); print(f"H2D 720 MB {name}: {t*1e3:.2f} ms = {720*MB/t/1e9:.1f} GB/s")
