#!/usr/bin/env python
"""NEXT-3: B200 crossover sweep of the paper's dense/sparse rule
on threshold matrices (Figs. 7-9): one community of M oscillators,
each pair connected with probability 1 - p (the paper's "z > p" threshold),
p in {0.01, 0.1, 0.3, 0.5, 0.7, 0.9, 0.99}.  For every p the same graph is
planned three ways — forced precomputed sums + complement lists
(dense_threshold = 1), forced direct summation (dense_threshold = 0, plain
CSR) and the paper's rule (precompute iff zeros < ones) — and one
kur_rhs evaluation is timed with CUDA events (median of R repetitions).

Reading R24: the paper draws every entry independently (an
asymmetric matrix); kurgen's generator is the symmetric SBM with one
community.  The stored-entry counts and hence the costs are the same in
expectation (M(M-1)·min(p, 1-p)), symmetry is not used by either summation.

  python tools/crossover.py [--m 16384] [--reps 20] > profiles/r01/crossover.jsonl
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

MODES = {"precompute": 1.0, "direct": 0.0, "rule": -1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=16384)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ps", default="0.01,0.1,0.3,0.5,0.7,0.9,0.99")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for p in (float(x) for x in args.ps.split(",")):
        inst = kurgen.sbm([args.m], [[1.0 - p]], 2102071670 + 300, K=1.0, permute=False, name=f"threshold-p{p}")
        # splay phases of P:588 (theta_m = 2 pi m / M) as in the paper's count experiments
        theta = torch.tensor(2.0 * np.pi * np.arange(1, args.m + 1) / args.m, dtype=torch.float64, device=dev)
        omega = torch.zeros(args.m, dtype=torch.float64, device=dev)
        ref = None
        for mode, thr in MODES.items():
            g = kur.graph_build(inst, dense_threshold=thr)
            th, om = g.to_internal(theta), g.to_internal(omega)
            out = kur.rhs(g, th, om, 1.0)
            for _ in range(3):
                kur.rhs(g, th, om, 1.0, out=out)
            ts = []
            for _ in range(args.reps):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                kur.rhs(g, th, om, 1.0, out=out)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            f = g.to_user(out).cpu().numpy()
            if ref is None:
                ref = f
            info = g.info
            print(json.dumps({
                "p": p, "density": 1.0 - p, "M": args.m, "mode": mode, "rhs_us": 1e3 * float(np.median(ts)),
                "n_idx": int(info["n_idx"]), "nnz": int(info["nnz"]), "dense_blocks": int(info["n_dense_blocks"]),
                "sparse_blocks": int(info["n_sparse_blocks"]), "bytes_per_rhs": int(info["bytes_per_rhs"]),
                "max_abs_diff_vs_first_mode": float(np.max(np.abs(f - ref))),
            }), flush=True)
            g.close()


if __name__ == "__main__":
    main()
