"""Write tests/golden/cfg<k>_oracle_trajectory_full.npz for a configured trajectory —
calls ONLY oracle/ and kurgen/ (test infrastructure; no value comes from the CUDA path).

  python tools/make_golden.py 4      # config 4: 200 RK4 steps, oracle matvec mode (O(nnz))

Stores theta after nsteps on a fixed sample of rows, r e^{i psi} at every step, the
instance SHA-256 (the test refuses another instance) and nsteps.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import kurgen  # noqa: E402
import oracle  # noqa: E402


def main(k):
    t0 = time.time()
    inst = kurgen.config(k)
    og = oracle.Graph(inst)
    th, _, rt = oracle.rk4(og, inst.theta0, inst.omega, inst.K, inst.h, inst.nsteps, 1, mode="matvec")
    rows = np.unique((kurgen.raw_bits(k, 11, 8192) % np.uint64(inst.n)).astype(np.int64))
    out = os.path.join(ROOT, "tests", "golden", f"cfg{k}_oracle_trajectory.npz")
    np.savez_compressed(out, sha256=inst.sha256(), nsteps=inst.nsteps, rows=rows, theta_final=th[rows],
                        r_trace=rt)
    print(f"wrote {out} ({inst.nsteps} steps, {rows.size} rows) in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main(int(sys.argv[1]))
