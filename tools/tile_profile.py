#!/usr/bin/env python
"""Per-tile phase breakdown of one k_stage launch (tooling).  Needs the
instrumented library: `make prof` (writes libkur_prof.so beside the product library).

  python tools/tile_profile.py [--config 5]
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["KUR_LIB"] = os.path.join(ROOT, "paper_2102_07167_b200", "libkur_prof.so")
import kurgen  # noqa: E402
from paper_2102_07167_b200 import kur  # noqa: E402

STRIDE = 192


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--hot-min", type=int, default=0)
    args = ap.parse_args()
    attach = kur._lib.kur_prof_attach
    attach.argtypes = [ctypes.c_void_p]
    inst = kurgen.config(args.config)
    g = kur.graph_build(inst, tile_rows=args.tile_rows, hot_min=args.hot_min)
    th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
    om = g.to_internal(torch.from_numpy(inst.omega).cuda())
    nt = int(g.info["n_tiles"])
    buf = torch.zeros(nt * STRIDE, dtype=torch.int64, device="cuda")
    kur.step(g, th, om, inst.K, inst.h, 2)
    attach(ctypes.c_void_p(buf.data_ptr()))
    kur.step(g, th, om, inst.K, inst.h, 1)
    torch.cuda.synchronize()
    attach(None)
    P = buf.view(nt, STRIDE).cpu().numpy().astype(np.float64)
    t0, t25, t26 = P[:, 0], P[:, 25], P[:, 26]
    nhot, nparts, nrem = P[:, 27].astype(int), P[:, 28].astype(int), P[:, 29].astype(int)
    tot = t26 - t0
    wait = np.zeros(nt); hot = np.zeros(nt); rem = np.zeros(nt); imb = np.zeros(nt)
    for t in range(nt):
        for p in range(min(nrem[t] + nhot[t], 8)):
            wb, we, pe = P[t, 1 + 3 * p], P[t, 2 + 3 * p], P[t, 3 + 3 * p]
            wf = P[t, 32 + 16 * p: 48 + 16 * p]
            wait[t] += we - wb
            (hot if p < nhot[t] else rem)[t] += pe - we  # the inline remote part runs last
            imb[t] += pe - wf.mean()
    fin = t26 - t25
    g0, g1, g2 = P[:, 160], P[:, 161], P[:, 162]
    t_first = g0.min()
    fin_end = g2[g2 > 0].max() if np.any(g2 > 0) else float("nan")
    print(f"global timeline (us from the first CTA start): last CTA start {(g0.max() - t_first) / 1e3:.2f}, "
          f"median tile done {(np.median(g1) - t_first) / 1e3:.2f}, last tile done {(g1.max() - t_first) / 1e3:.2f}, "
          f"finish done {(fin_end - t_first) / 1e3:.2f}")
    q = np.percentile(tot, [50, 90, 99, 100])
    print(f"tile cycles p50 {q[0]:.0f} p90 {q[1]:.0f} p99 {q[2]:.0f} max {q[3]:.0f}; "
          f"remote part p50 {np.percentile(rem, 50):.0f} max {rem.max():.0f}; hot p50 {np.percentile(hot, 50):.0f} "
          f"max {hot.max():.0f}")
    print(f"cfg{args.config}: {nt} tiles, rows/tile {g.info['rows_per_tile']}, parts/tile {nparts.mean():.2f} "
          f"(hot {nhot.mean():.2f})")
    print(f"mean cycles per tile: total {tot.mean():.0f}")
    for name, v in (("window wait", wait), ("hot parts (incl. tail)", hot), ("remote parts (incl. tail)", rem),
                    ("  of which barrier tail (part end - mean warp finish)", imb), ("finalize", fin)):
        print(f"  {name:52s} {v.mean():10.0f}  {v.mean() / tot.mean():6.3f}")
    g.close()


if __name__ == "__main__":
    main()
