#!/usr/bin/env python
"""Strong-scaling model of config 5 from measured per-rank kernel times (tooling, one GPU).

Every box of this run has one GPU, so bench.py --gpus N cannot be timed.  This tool builds the
world-G rank handles of config 5 in one process (kur_group_*: the same plans, kernels and phases as
the NCCL path, with the per-stage all-gather done by device copies) and times every rank's kernels
with CUDA events.  Each rank's kernels run alone on the GPU, as they would on that rank's own
B200, so per stage and rank:  compute_r = phase A (own-community windows, overlaps the previous
exchange) + k_remote + phase B (the rest + the fused RK epilogue).  The model
T_G = max_r compute_r assumes the exchange of stage s (all-gather of ~8 B per row + unpack +
fixed-order finish, on a priority stream) hides behind phase A of stage s+1; it reports the
exchange volume per rank next to phase A so the assumption can be checked against NVLink rates.

  python tools/scaling_model.py [--worlds 2 4 8] [--steps 4]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import kurgen  # noqa: E402
from paper_2102_07167_b200 import kur  # noqa: E402


def per_stage(g, steps):
    t = kur.timing_read(g)
    n = 4 * steps
    return {"stage_ms": t["stage_ms"] / n, "remote_ms": t["remote_ms"] / n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    inst = kurgen.config(args.config)
    dev = "cuda:0"
    g1 = kur.graph_build(inst)
    th = g1.to_internal(torch.from_numpy(inst.theta0).to(dev))
    om = g1.to_internal(torch.from_numpy(inst.omega).to(dev))
    a = th.clone()
    kur.step(g1, a, om, inst.K, inst.h, 2)
    kur.timing(g1, True)
    kur.step(g1, a, om, inst.K, inst.h, args.steps)
    torch.cuda.synchronize()
    t1 = per_stage(g1, args.steps)
    T1 = t1["stage_ms"] + t1["remote_ms"]
    g1.close()
    out = {"config": inst.name, "T1_stage_ms": T1, "worlds": []}
    for G in args.worlds:
        gs = kur.group_build(inst, G)
        ths = [th[g.row_begin:g.row_end].clone() for g in gs]
        oms = [om[g.row_begin:g.row_end].clone() for g in gs]
        kur.group_step(gs, ths, oms, inst.K, inst.h, 2)
        for g in gs:
            kur.timing(g, True)
        kur.group_step(gs, ths, oms, inst.K, inst.h, args.steps)
        torch.cuda.synchronize()
        ranks = [per_stage(g, args.steps) for g in gs]
        comp = [r["stage_ms"] + r["remote_ms"] for r in ranks]
        TG = max(comp)
        xbytes = 8 * inst.n * (G - 1) / G  # theta of the other ranks' rows received per rank per stage
        out["worlds"].append({
            "G": G, "rank_compute_ms": comp, "T_G_model_ms": TG, "efficiency_model": T1 / (G * TG),
            "rows_per_rank": [g.n_local for g in gs],
            "exchange_bytes_received_per_rank": xbytes,
            "exchange_ms_at_400GBps": xbytes / 400e9 * 1e3})
        print(f"G={G}: per-rank compute per stage {np.round(comp, 4).tolist()} ms, model T_G {TG:.4f} ms, "
              f"efficiency {T1 / (G * TG):.3f}; exchange {xbytes / 1e6:.1f} MB/rank "
              f"(~{xbytes / 400e9 * 1e6:.0f} us at 400 GB/s)", flush=True)
        for g in gs:
            g.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
