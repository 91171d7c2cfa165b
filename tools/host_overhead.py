"""Host-side cost of one rd.inverse_dynamics call (small batch): Python binding vs C ABI."""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth, paper_1609_04493_b200 as rd
n, B = 8, 16
m = rd.Model.from_robot(synth.random_chain(n, 1008), synth.GRAVITY_Z)
q, qd, qdd = (torch.rand(n, B, dtype=torch.float64, device="cuda") for _ in range(3))
out = torch.empty_like(q)
for strat in ("warp_scan", "reverse"):
    m.set_strategy(strat)
    for _ in range(100):
        rd.inverse_dynamics(m, q, qd, qdd, out)
    torch.cuda.synchronize()
    N = 2000
    t0 = time.perf_counter()
    for _ in range(N):
        rd.inverse_dynamics(m, q, qd, qdd, out)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    L = rd.lib(); s = torch.cuda.current_stream().cuda_stream
    a, b_, c, o = q.data_ptr(), qd.data_ptr(), qdd.data_ptr(), out.data_ptr()
    t3 = time.perf_counter()
    for _ in range(N):
        L.rd_inverse_dynamics_f64(m.handle, B, a, b_, c, o, s)
    t4 = time.perf_counter()
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"{strat}: python binding {1e6*(t1-t0)/N:.1f} us/call (incl. drain {1e6*(t2-t0)/N:.1f}); "
          f"raw C ABI {1e6*(t4-t3)/N:.1f} us/call (incl. drain {1e6*(t5-t3)/N:.1f})")
