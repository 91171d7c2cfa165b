"""Measured host<->device copy bandwidth (pinned buffers) on this box: the ceiling of the
e2e host-buffer path (720 MB H2D + 240 MB D2H per C3 step).  Development aid."""
import time
import torch

MB = 1 << 20
h_in = torch.empty(720 * MB // 8, dtype=torch.float64).pin_memory()
h_out = torch.empty(240 * MB // 8, dtype=torch.float64).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty_like(h_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


t_h2d = timed(lambda: d_in.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_out, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


t_both = timed(both)
print(f"H2D {720 * MB / t_h2d / 1e9:.1f} GB/s  D2H {240 * MB / t_d2h / 1e9:.1f} GB/s  "
      f"H2D+D2H concurrent {t_both * 1e3:.2f} ms per C3-sized step (720 MB in, 240 MB out) "
      f"-> e2e ceiling {1e6 / t_both:.3e} evals/s at n = 30")
