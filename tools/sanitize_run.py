#!/usr/bin/env python
"""Small workload touching every kernel path, for compute-sanitizer:

  compute-sanitizer --tool memcheck|racecheck|synccheck|initcheck python tools/sanitize_run.py

k_small (single-CTA trajectory), multi-tile k_stage with hot windows and inline remote parts,
the k_remote pass, every integrator, the potential, the order parameter, adaptive RK4, and the
sharded group path with both exchanges (device copies and fused peer stores)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import kurgen  # noqa: E402
from paper_2102_07167_b200 import kur  # noqa: E402


def run(inst, **kw):
    g = kur.graph_build(inst, **kw)
    th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    kur.rhs(g, th, om, inst.K)
    kur.step(g, th.clone(), om, inst.K, inst.h, 2, 1, check=True)
    for m in ("euler", "heun", "implicit_midpoint"):
        kur.step_method(g, m, th.clone(), om, inst.K, inst.h, 2, 1, check=True)
    kur.potential(g, th, om, inst.K)
    kur.order_parameter(g, th, local=True)
    kur.integrate_adaptive(g, th.clone(), om, inst.K, 0.02, 0.01, atol=1e-8, rtol=1e-8)
    torch.cuda.synchronize()
    g.close()


def main():
    small = kurgen.sbm([300, 200], [[0.9, 0.05], [0.05, 0.7]], 1, K=2.0, h=0.01)           # k_small
    mid = kurgen.sbm([3000, 2500, 1200, 9], np.array([[0.97, 0.002, 0.01, 0.0], [0.002, 0.95, 0.003, 0.0],
                                                      [0.01, 0.003, 0.2, 0.1], [0.0, 0.0, 0.1, 0.5]]), 2,
                     K=3.0, h=0.01)
    run(small)
    run(mid, tile_rows=512)                          # hot windows + inline remote part
    run(mid, tile_rows=512, remote_pass=True)        # k_remote pass
    run(mid, hot_min=1 << 30)                        # everything remote
    for peer in (False, True):                       # sharded path, world 3 (device copies / peer stores)
        gs = kur.group_build(mid, 3, peer_exchange=peer, tile_rows=512)
        full = gs[0].to_internal(torch.from_numpy(mid.theta0).cuda())
        omf = gs[0].to_internal(torch.from_numpy(mid.omega).cuda())
        ths = [full[g.row_begin:g.row_end].clone() for g in gs]
        oms = [omf[g.row_begin:g.row_end].clone() for g in gs]
        kur.group_rhs(gs, ths, oms, mid.K)
        kur.group_step(gs, ths, oms, mid.K, mid.h, 2, 1)
        kur.group_step_method(gs, "implicit_midpoint", ths, oms, mid.K, mid.h, 2, 1)
        torch.cuda.synchronize()
        for g in gs:
            g.close()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
