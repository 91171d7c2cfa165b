import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth, paper_1609_04493_b200 as rd
cfg = synth.CONFIGS["C3"]
q, qd, qdd = synth.states(cfg["seed"], 30, 0, 1_000_000)
pq, pqd, pqdd = (torch.from_numpy(x).pin_memory() for x in (q, qd, qdd))
out = torch.empty_like(pq).pin_memory()
m = rd.Model.from_robot(synth.robot_for(cfg), cfg["gravity"])
rd.inverse_dynamics_host(m, pq, pqd, pqdd, out)
t0 = time.perf_counter()
for _ in range(5):
    rd.inverse_dynamics_host(m, pq, pqd, pqdd, out)
dt = (time.perf_counter() - t0) / 5
print(f"chunk={os.environ.get('RD_HOST_CHUNK_MB')} e2e {dt*1e3:.2f} ms  {1e6/dt:.3e} evals/s  H2D {720e6/dt/1e9:.1f} GB/s")
# raw copy bandwidth reference
x = torch.empty(90_000_000, dtype=torch.float64).pin_memory(); y = torch.empty_like(x, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); y.copy_(x, non_blocking=True); torch.cuda.synchronize()
print(f"raw H2D {720e6/(time.perf_counter()-t0)/1e9:.1f} GB/s")
