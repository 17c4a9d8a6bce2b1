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
