"""Multi-process NCCL path: 2 ranks, one process per GPU, exactly as
bench.py --gpus 2 runs it.  Needs >= 2 visible GPUs (skipped otherwise: every gpurun box
and the driver's round-end box have one).  Each rank builds its shard with an NCCL
communicator; the per-stage exchange is ncclAllGather or the fused peer-store exchange
(CUDA IPC over NVLink).  Results must be BITWISE equal to world 1, for RK4, one NEXT-4
method (Heun) and the end-to-end host-buffer call."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inst():
    import kurgen
    return kurgen.sbm([3000, 500, 2000, 4100, 77], np.array(
        [[0.95, 0.01, 0.0, 0.6, 0.0], [0.01, 0.3, 0.02, 0.0, 0.0], [0.0, 0.02, 0.97, 0.001, 0.1],
         [0.6, 0.0, 0.001, 0.99, 0.0], [0.0, 0.0, 0.1, 0.0, 0.5]]), 23, K=3.0, h=0.01)


def _worker(rank, port, peer, q):
    import sys
    sys.path.insert(0, ROOT)
    try:
        import torch.distributed as dist
        from paper_2102_07167_b200 import kur
        torch.cuda.set_device(rank)
        dev = torch.device(f"cuda:{rank}")
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=WORLD,
                                device_id=dev)
        inst = _inst()
        obj = [kur.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = kur.graph_build(inst, device=rank, dist=(rank, WORLD, obj[0], kur.DIST_PEER_EXCHANGE if peer else 0))
        assert g.info["world"] == WORLD and g.info["peer_exchange"] == int(peer)
        th_full = g.to_internal(torch.from_numpy(inst.theta0).to(dev))
        om_full = g.to_internal(torch.from_numpy(inst.omega).to(dev))
        th = g.local(th_full).clone()
        om = g.local(om_full).clone()
        f = kur.rhs(g, th, om, inst.K)
        th_rk = th.clone()
        rt_rk = kur.step(g, th_rk, om, inst.K, inst.h, 6, 1, check=True)
        th_he = th.clone()
        rt_he = kur.step_method(g, "heun", th_he, om, inst.K, inst.h, 6, 1, check=True)
        th_host = th.cpu().pin_memory()
        kur.step(g, th_host, om, inst.K, inst.h, 6, 1)  # host-buffer (end-to-end) call at world 2
        torch.cuda.synchronize()
        parts = {k: [None] * WORLD for k in ("f", "rk", "he", "host")}
        for k, v in (("f", f), ("rk", th_rk), ("he", th_he), ("host", th_host)):
            dist.all_gather_object(parts[k], v.cpu().numpy())
        if rank == 0:  # world 1 on this GPU
            g1 = kur.graph_build(inst, device=0)
            t1 = g1.to_internal(torch.from_numpy(inst.theta0).to(dev))
            o1 = g1.to_internal(torch.from_numpy(inst.omega).to(dev))
            f1 = kur.rhs(g1, t1, o1, inst.K).cpu().numpy()
            a = t1.clone()
            r1 = kur.step(g1, a, o1, inst.K, inst.h, 6, 1)
            b = t1.clone()
            r2 = kur.step_method(g1, "heun", b, o1, inst.K, inst.h, 6, 1)
            torch.cuda.synchronize()
            assert np.array_equal(np.concatenate(parts["f"]), f1), "rhs"
            assert np.array_equal(np.concatenate(parts["rk"]), a.cpu().numpy()), "rk4"
            assert np.array_equal(np.concatenate(parts["he"]), b.cpu().numpy()), "heun"
            assert np.array_equal(np.concatenate(parts["host"]), a.cpu().numpy()), "host buffers"
            assert torch.equal(rt_rk, r1) and torch.equal(rt_he, r2), "r_trace"
            g1.close()
        g.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("peer", [False, True])
def test_nccl_two_ranks_bitwise_equal_world1(peer):
    if torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs (this box has {torch.cuda.device_count()})")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, peer, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(WORLD))
    for p in procs:
        p.join(timeout=60)
    for r in range(WORLD):
        assert res[r] == "ok", res[r]


def test_bench_two_gpus_prints_one_line():
    """bench.py --gpus 2 (self-launched torchrun, NCCL) prints one JSON line with n_gpus 2 and an
    end-to-end number; NCCL's INIT lines go to stderr."""
    if torch.cuda.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs")
    import json
    import subprocess
    import sys
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "3",
                          "--steps", "5", "--warmup", "3", "--no-cpu"], capture_output=True, text=True, env=env,
                         timeout=1200)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["e2e"]["value"] > 0
    assert "nranks 2" in out.stderr or "nRanks 2" in out.stderr
