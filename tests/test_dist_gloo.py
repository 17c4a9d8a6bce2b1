"""Multi-process host-side logic of the sharded path (world_size 2, gloo, CPU).

Each process builds ITS rank's block plan independently (kur_plan_build, no
GPU), exactly as kur_graph_build does on a GPU box.  Over gloo the ranks then
check that (1) they agree on the shard boundaries, the permutation and the
dense-block lists, (2) their shards tile the rows and, decoded, reproduce the
world-1 plan row by row, and (3) the packed all-gather layout used per RK
stage ([stage phases of the shard | tile partials], padded to the largest
shard) reconstructs the global vectors on every rank.
"""
import hashlib
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inst(kind="sbm"):
    import kurgen
    if kind == "one_community":  # a single dense community: shards split it between tiles
        rng = np.random.default_rng(11)
        n = 2600
        A = (rng.random((n, n)) < 0.96).astype(np.uint8)
        A = np.triu(A, 1)
        A = A + A.T
        return kurgen.from_dense(A, np.zeros(n, np.int64), kind="zeros")
    return kurgen.sbm([900, 300, 1200, 700, 64, 1], np.array(
        [[0.95, 0.01, 0.0, 0.0, 0.3, 0.0], [0.01, 0.3, 0.02, 0.0, 0.0, 0.0], [0.0, 0.02, 0.97, 0.6, 0.0, 0.0],
         [0.0, 0.0, 0.6, 0.99, 0.0, 0.0], [0.3, 0.0, 0.0, 0.0, 0.5, 0.0], [0.0] * 6]), 31)


def _rows(plan):
    out = {}
    for lj in range(plan["n_local"]):
        s, e = plan["row_ptr"][lj], plan["row_ptr"][lj + 1]
        key = sorted(zip(plan["cols"][s:e].tolist(), plan["neg"][s:e].tolist()))
        out[plan["row_begin"] + lj] = key
    return out


def _worker(rank, world, port, q, kind="sbm"):
    import sys
    sys.path.insert(0, ROOT)
    try:
        from paper_2102_07167_b200 import kur
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        inst = _inst(kind)
        tr = 256 if kind == "one_community" else 0
        plan = kur.plan_export(inst, rank=rank, world=world, tile_rows=tr)
        meta = dict(rank=rank, row_begin=plan["row_begin"], n_local=plan["n_local"],
                    shard=plan["shard_row0"].tolist(),
                    perm=hashlib.sha256(plan["perm"].tobytes()).hexdigest(),
                    D=hashlib.sha256(plan["D_ptr"].tobytes() + plan["D_idx"].tobytes()).hexdigest())
        metas = [None] * world
        dist.all_gather_object(metas, meta)
        for m in metas:
            assert m["shard"] == metas[0]["shard"] and m["perm"] == metas[0]["perm"] and m["D"] == metas[0]["D"]
            assert m["row_begin"] == m["shard"][m["rank"]]
            assert m["row_begin"] + m["n_local"] == m["shard"][m["rank"] + 1]
        # decoded rows of this shard == the world-1 plan's rows
        ref = _rows(kur.plan_export(inst, tile_rows=tr))
        if kind == "one_community":
            assert 0 < plan["n_local"] < inst.n  # both ranks hold rows of the one community
        mine = _rows(plan)
        for j, ents in mine.items():
            assert ents == ref[j], j
        # packed exchange layout: [theta of the shard, padded to xrows | partials]
        shard = metas[0]["shard"]
        xrows = max(shard[r + 1] - shard[r] for r in range(world))
        theta_global = np.sin(np.arange(inst.n) * 0.37) + np.arange(inst.n) * 1e-3
        send = np.zeros(xrows, np.float64)
        send[: plan["n_local"]] = theta_global[plan["row_begin"]: plan["row_begin"] + plan["n_local"]]
        recv = [torch.zeros(xrows, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, torch.from_numpy(send))
        rebuilt = np.concatenate([recv[r].numpy()[: shard[r + 1] - shard[r]] for r in range(world)])
        assert np.array_equal(rebuilt, theta_global)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("world,kind", [(2, "sbm"), (2, "one_community")])
def test_sharded_plans_agree_over_gloo(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kind)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r] == "ok", res[r]


def test_bench_gpus_n_launches_n_ranks():
    """`bench.py --gpus 2` without a torchrun environment launches 2 ranks itself (torch.distributed.run,
    127.0.0.1) and prints exactly one JSON line with n_gpus 2 (reference arm: rank 0 runs the oracle on
    the host, the other rank exits 0; no GPU needed)."""
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "1", "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_bench_rejects_gpus_world_mismatch():
    import subprocess
    import sys
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--config", "1"], capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr
