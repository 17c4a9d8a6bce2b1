"""Write tests/golden/cfg5_oracle_trajectory.npz — calls ONLY oracle/ and kurgen/.

Config 5 (N = 2^22) is too large for the oracle to integrate inside the GPU
test run, so its reference trajectory (oracle matvec mode, O(nnz), no
block sums) is computed once here and stored: theta after 10 RK4 steps on a
fixed sample of rows, and the complex order parameter at steps 0..10.  The
instance SHA-256 is stored so the test refuses a different instance.
~10 minutes on 8 cores.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import kurgen  # noqa: E402
import oracle  # noqa: E402


def main():
    t0 = time.time()
    inst = kurgen.config(5)
    print(f"generated in {time.time() - t0:.1f}s, sha {inst.sha256()[:16]}", flush=True)
    og = oracle.Graph(inst)
    t0 = time.time()
    th, th10, rt = oracle.rk4(og, inst.theta0, inst.omega, inst.K, inst.h, 10, 1, mode="matvec")
    print(f"oracle 10 RK4 steps in {time.time() - t0:.1f}s", flush=True)
    rows = np.unique(np.concatenate([
        (kurgen.raw_bits(55, 9, 8192) % np.uint64(inst.n)).astype(np.int64),
        np.flatnonzero(inst.community == 7)[:2048].astype(np.int64),
    ]))
    out = os.path.join(ROOT, "tests", "golden", "cfg5_oracle_trajectory.npz")
    np.savez_compressed(out, sha256=np.array(inst.sha256()), rows=rows, theta10=th10[rows], r_trace=rt,
                        note=np.array("oracle matvec RK4 (h=0.01) of kurgen.config(5); written by "
                                      "tools/make_golden_cfg5.py (oracle/ + kurgen/ only)"))
    print("wrote", out, rows.size, "rows")


if __name__ == "__main__":
    main()
