"""Sharded path on one GPU: world = 2/3/4 rank handles run
the same kernels as the NCCL path, with the per-stage all-gather done by
device copies (kur_group_*).  Results must be BITWISE equal to world = 1
(communities are never split, tile partials are reduced in a fixed order)."""
import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import close

pytestmark = pytest.mark.gpu


def _instances():
    yield "sbm5", kurgen.sbm([3000, 500, 2000, 4100, 77], np.array(
        [[0.95, 0.01, 0.0, 0.6, 0.0], [0.01, 0.3, 0.02, 0.0, 0.0], [0.0, 0.02, 0.97, 0.001, 0.1],
         [0.6, 0.0, 0.001, 0.99, 0.0], [0.0, 0.0, 0.1, 0.0, 0.5]]), 23, K=3.0, h=0.01)
    yield "cfg3", kurgen.config(3)


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("remote_pass", [None, True])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_group_bitwise_equals_single(world, remote_pass, peer):
    for name, inst in _instances():
        g1 = kur.graph_build(inst, remote_pass=remote_pass)
        dev = "cuda:0"
        th_full = g1.to_internal(torch.from_numpy(inst.theta0).to(dev))
        om_full = g1.to_internal(torch.from_numpy(inst.omega).to(dev))
        f1 = kur.rhs(g1, th_full, om_full, inst.K)
        th1 = th_full.clone()
        rt1 = kur.step(g1, th1, om_full, inst.K, inst.h, 6, 1)

        gs = kur.group_build(inst, world, remote_pass=remote_pass, peer_exchange=peer)
        assert all(np.array_equal(g.perm, g1.perm) for g in gs)
        bounds = [(g.row_begin, g.row_end) for g in gs]
        assert bounds[0][0] == 0 and bounds[-1][1] == inst.n
        assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
        ths = [th_full[g.row_begin:g.row_end].clone() for g in gs]
        oms = [om_full[g.row_begin:g.row_end].clone() for g in gs]
        fs = kur.group_rhs(gs, ths, oms, inst.K)
        assert torch.equal(torch.cat(fs), f1), (name, world, "rhs")
        rts = kur.group_step(gs, ths, oms, inst.K, inst.h, 6, 1)
        torch.cuda.synchronize()
        assert all(g.refresh_info()["peer_exchange"] == int(peer) for g in gs)
        assert torch.equal(torch.cat(ths), th1), (name, world, "theta after 6 steps")
        for rt in rts:
            assert torch.equal(rt, rt1), (name, world, "r_trace")
        for g in gs:
            g.close()
        g1.close()


def test_group_parity_with_oracle():
    name, inst = next(_instances())
    gs = kur.group_build(inst, 3)
    dev = "cuda:0"
    th_full = gs[0].to_internal(torch.from_numpy(inst.theta0).to(dev))
    om_full = gs[0].to_internal(torch.from_numpy(inst.omega).to(dev))
    ths = [th_full[g.row_begin:g.row_end].clone() for g in gs]
    oms = [om_full[g.row_begin:g.row_end].clone() for g in gs]
    rts = kur.group_step(gs, ths, oms, inst.K, inst.h, 10, 1)
    got = np.empty(inst.n)
    got[gs[0].perm] = torch.cat(ths).cpu().numpy()
    th_ref, th10_ref, rt_ref = oracle.rk4(oracle.Graph(inst), inst.theta0, inst.omega, inst.K, inst.h, 10, 1,
                                          mode="naive")
    ok, err = close(got, th10_ref)
    assert ok, err
    rt = rts[0].cpu().numpy()
    d = np.abs(rt[:, 0] * np.exp(1j * rt[:, 1]) - rt_ref[:, 0] * np.exp(1j * rt_ref[:, 1]))
    assert d.max() <= 1e-9


def test_group_handle_alone_is_refused():
    name, inst = next(_instances())
    gs = kur.group_build(inst, 2)
    th = torch.zeros(gs[0].n_local, dtype=torch.float64, device="cuda:0")
    with pytest.raises(kur.KurError) as e:
        kur.step(gs[0], th, th.clone(), 1.0, 0.01, 1)
    assert e.value.status == 10


def _group_vs_single(inst, world, steps=4, method="rk4", **kw):
    """world-rank group (one device) against world 1: RHS, `steps` steps and r(t), bitwise."""
    g1 = kur.graph_build(inst, **kw)
    dev = "cuda:0"
    th_full = g1.to_internal(torch.from_numpy(inst.theta0).to(dev))
    om_full = g1.to_internal(torch.from_numpy(inst.omega).to(dev))
    f1 = kur.rhs(g1, th_full, om_full, inst.K)
    th1 = th_full.clone()
    rt1 = kur.step_method(g1, method, th1, om_full, inst.K, inst.h, steps, 1)
    gs = kur.group_build(inst, world, **kw)
    ths = [th_full[g.row_begin:g.row_end].clone() for g in gs]
    oms = [om_full[g.row_begin:g.row_end].clone() for g in gs]
    fs = kur.group_rhs(gs, ths, oms, inst.K)
    rts = kur.group_step_method(gs, method, ths, oms, inst.K, inst.h, steps, 1)
    torch.cuda.synchronize()
    ok = (torch.equal(torch.cat(fs), f1), torch.equal(torch.cat(ths), th1), all(torch.equal(r, rt1) for r in rts))
    bounds = [(g.row_begin, g.row_end) for g in gs]
    for g in gs:
        g.close()
    g1.close()
    return ok, bounds


@pytest.mark.parametrize("case", ["sbm_2x1000", "complete_20000", "one_community_9000"])
@pytest.mark.parametrize("world", [2, 3])
def test_group_bitwise_world_independent_tiles(case, world):
    """The world-independent tile rule (builder.cpp) makes ANY world size bitwise equal to world 1,
    including graphs the round-1 rule tiled differently per world (a small SBM: tiny-graph tiles;
    a complete graph: entry-free tiles sized by n / world) and a single community split between
    ranks at tile boundaries (phase A then only sums the windows inside the rank's rows)."""
    if case == "sbm_2x1000":
        inst = kurgen.sbm([1000, 1000], np.array([[0.02, 0.02], [0.02, 0.02]]), 5, K=2.0, h=0.01)
    elif case == "complete_20000":
        inst = kurgen.complete_graph(20000, 9, K=3.0, h=0.01)
    else:
        rng = np.random.default_rng(3)
        n = 9000
        A = (rng.random((n, n)) < 0.97).astype(np.uint8)
        A = np.triu(A, 1)
        A = A + A.T
        inst = kurgen.from_dense(A, np.zeros(n, np.int64), kind="zeros", seed=4, K=2.0, h=0.01)
    for method in ("rk4", "heun"):
        ok, bounds = _group_vs_single(inst, world, method=method)
        assert all(ok), (case, world, method, ok)
    if case != "sbm_2x1000":  # one community: every rank holds rows
        assert all(b > a for a, b in bounds), bounds


@pytest.mark.parametrize("world", [1, 2])
def test_remote_modes_bitwise(world, monkeypatch):
    """The remote part summed by the k_remote pass (KUR_REMOTE_MODE=0), by one warp of the stage kernel
    with TMA 16-byte gathers (1), LDG gathers (2) or TMA tile::gather4 (3): the same bits (world 2:
    phase B with the remote warp)."""
    inst = kurgen.sbm([4000, 3000, 2500, 2600], np.array(
        [[0.97, 0.01, 0.002, 0.0], [0.01, 0.9, 0.0, 0.01], [0.002, 0.0, 0.98, 0.003], [0.0, 0.01, 0.003, 0.95]]),
        41, K=3.0, h=0.01)
    res = []
    for mode in ("0", "1", "2", "3"):
        monkeypatch.setenv("KUR_REMOTE_MODE", mode)
        if world == 1:
            g = kur.graph_build(inst, remote_pass=True, tile_rows=512)
            assert g.info["remote_pass"] == 1
            th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
            om = g.to_internal(torch.from_numpy(inst.omega).cuda())
            f = kur.rhs(g, th, om, inst.K)
            rt = kur.step(g, th, om, inst.K, inst.h, 5, 1)
            res.append((f, th, rt))
            g.close()
        else:
            ok, _ = _group_vs_single(inst, world, steps=5, remote_pass=True, tile_rows=512)
            assert all(ok), (mode, ok)
    if world == 1:
        for f, th, rt in res[1:]:
            assert torch.equal(f, res[0][0]) and torch.equal(th, res[0][1]) and torch.equal(rt, res[0][2])


def test_config5_world8_bitwise():
    """Config 5 (the scaling workload) split over 8 rank handles on one device, as bench.py --gpus 8
    shards it (32 whole communities per rank): RHS, 2 RK4 steps and r(t) bitwise equal to world 1."""
    inst = kurgen.config(5)
    ok, bounds = _group_vs_single(inst, 8, steps=2)
    assert all(ok), ok
    assert len(bounds) == 8 and all(b - a == inst.n // 8 for a, b in bounds), bounds


@pytest.mark.parametrize("world", [1, 2])
def test_concurrent_inline_remote_bitwise(world, monkeypatch):
    """The inline remote part run concurrently with the hot windows on warps [k, 16) (KUR_CONC_REMOTE=k,
    k_stage<..., CR>) gives the bits of the sequential inline part and of the k_remote pass."""
    inst = kurgen.sbm([3000, 2000, 2500, 1200], np.array(
        [[0.95, 0.004, 0.003, 0.002], [0.004, 0.97, 0.003, 0.005], [0.003, 0.003, 0.9, 0.004],
         [0.002, 0.005, 0.004, 0.96]]), 43, K=3.0, h=0.01)
    ref = None
    for mode, rp in (("0", False), ("8", False), ("4", False), ("12", False), ("0", True)):
        monkeypatch.setenv("KUR_CONC_REMOTE", mode)
        if world == 1:
            g = kur.graph_build(inst, remote_pass=rp, tile_rows=256)
            th = g.to_internal(torch.from_numpy(inst.theta0).cuda())
            om = g.to_internal(torch.from_numpy(inst.omega).cuda())
            f = kur.rhs(g, th, om, inst.K)
            rt = kur.step(g, th, om, inst.K, inst.h, 5, 1)
            out = (f, th, rt)
            g.close()
            if ref is None:
                ref = out
            else:
                assert all(torch.equal(x, y) for x, y in zip(out, ref)), (mode, rp)
        else:
            ok, _ = _group_vs_single(inst, world, steps=4, remote_pass=rp, tile_rows=256)
            assert all(ok), (mode, rp, ok)
