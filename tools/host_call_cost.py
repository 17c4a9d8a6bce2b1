import time, torch, numpy as np, kurgen
from paper_2102_07167_b200 import kur
inst = kurgen.config(1)
g = kur.graph_build(inst)
th = g.to_internal(torch.from_numpy(inst.theta0).cuda()); om = g.to_internal(torch.from_numpy(inst.omega).cuda())
rt = torch.zeros((2, 2), dtype=torch.float64, device="cuda")
for _ in range(100): kur.step(g, th, om, inst.K, inst.h, 1, 1, r_trace=rt)
torch.cuda.synchronize()
for n in (1, 50):
    t0 = time.perf_counter()
    for _ in range(2000): kur.step(g, th, om, inst.K, inst.h, n, 1, r_trace=torch.zeros((n + 1, 2), dtype=torch.float64, device="cuda") if n > 1 else rt)
    torch.cuda.synchronize()
    print("nsteps", n, "us per call", (time.perf_counter() - t0) / 2000 * 1e6)
