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

os.environ.setdefault("KUR_REMOTE_SEQ", "1")  # per-rank kernels measured one after another (no cross-rank overlap)

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import kurgen  # noqa: E402
from paper_2102_07167_b200 import kur  # noqa: E402


def per_stage(g, steps):
    t = kur.timing_read(g)
    n = 4 * steps
    return {"stage_ms": t["stage_ms"] / n, "remote_ms": t["remote_ms"] / n, "phase_a_ms": t["phase_a_ms"] / n}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--worlds", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--remote-pass", default="auto", choices=["auto", "on", "off"])
    ap.add_argument("--tile-rows", type=int, default=0)
    args = ap.parse_args()
    rp = {"auto": None, "on": True, "off": False}[args.remote_pass]
    inst = kurgen.config(args.config)
    dev = "cuda:0"
    g1 = kur.graph_build(inst, tile_rows=args.tile_rows)
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
        gs = kur.group_build(inst, G, remote_pass=rp, tile_rows=args.tile_rows)
        ths = [th[g.row_begin:g.row_end].clone() for g in gs]
        oms = [om[g.row_begin:g.row_end].clone() for g in gs]
        kur.group_step(gs, ths, oms, inst.K, inst.h, 2)
        for g in gs:
            kur.timing(g, True)
        kur.group_step(gs, ths, oms, inst.K, inst.h, args.steps)
        torch.cuda.synchronize()
        ranks = [per_stage(g, args.steps) for g in gs]
        comp = [r["stage_ms"] + r["remote_ms"] for r in ranks]  # no overlap of k_remote
        comp_ov = [r["stage_ms"] for r in ranks]  # k_remote fully hidden behind phase A (exchange stream)
        ph_a = [r["phase_a_ms"] for r in ranks]
        ph_b = [r["stage_ms"] - r["phase_a_ms"] for r in ranks]
        rem = [r["remote_ms"] for r in ranks]
        print(f"G={G}: phase A {np.round(ph_a, 4).tolist()}  k_remote {np.round(rem, 4).tolist()}  "
              f"phase B {np.round(ph_b, 4).tolist()} ms per stage", flush=True)
        TG = max(comp)
        # on NCCL ranks k_remote runs on the exchange stream after the previous exchange (all-gather of the
        # other ranks' phases at ~400 GB/s received, unpack ~ one sincos + 16 B store per received row):
        # overlapped T = max(A, X + R) + B
        xms = (8 * inst.n * (G - 1) / G) / 400e9 * 1e3 + (inst.n * (G - 1) / G) * 24 / 3.0e12 * 1e3
        TGo = max(max(a, xms + r) + b for a, r, b in zip([r_["phase_a_ms"] for r_ in ranks],
                                                        [r_["remote_ms"] for r_ in ranks],
                                                        [r_["stage_ms"] - r_["phase_a_ms"] for r_ in ranks]))
        xbytes = 8 * inst.n * (G - 1) / G  # theta of the other ranks' rows received per rank per stage
        print(f"G={G}: k_remote on the exchange stream (exchange + unpack ~{xms * 1e3:.0f} us): model T_G "
              f"{TGo:.4f} ms, efficiency {T1 / (G * TGo):.3f}", flush=True)
        out["worlds"].append({"T_G_overlap_ms": TGo, "efficiency_overlap": T1 / (G * TGo),
            "G": G, "rank_compute_ms": comp, "phase_a_ms": ph_a, "phase_b_ms": ph_b, "k_remote_ms": rem,
            "T_G_model_ms": TG, "efficiency_model": T1 / (G * TG),
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
