"""GPU parity for NEXT-4: the paper's other one-step integrators (explicit
Euler P:303-306, Heun and implicit midpoint P:376) on the same localised-order-
parameter RHS, through kur_step_method, against oracle.step_method.  Tolerances
are BASELINE's north_star ones (theta after 10 steps: 1e-9 abs + 1e-12 rel;
complex r e^{i psi}: 1e-9)."""
import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import Run, close, complex_rpsi

pytestmark = pytest.mark.gpu

METHODS = ["euler", "heun", "implicit_midpoint"]


def _gpu(run, method, nsteps, record_every=1, h=None, **kw):
    th = run.theta_int.clone()
    rt = kur.step_method(run.g, method, th, run.omega_int, run.inst.K, run.inst.h if h is None else h, nsteps,
                         record_every, check=True, **kw)
    torch.cuda.synchronize()
    return run.user(th), rt.cpu().numpy()


def _check(inst, method, nsteps=10, mode="naive", **kw):
    run = Run(inst, **{k: v for k, v in kw.items() if k in ("dense_threshold", "tile_rows", "hot_min", "remote_pass")})
    fp = {k: v for k, v in kw.items() if k in ("fp_tol", "fp_max_iter")}
    th, rt = _gpu(run, method, nsteps, **fp)
    th_ref, rt_ref = oracle.step_method(oracle.Graph(inst), method, inst.theta0, inst.omega, inst.K, inst.h, nsteps,
                                        1, mode=mode, **fp)
    ok, err = close(th, th_ref)
    assert ok, (method, err)
    assert np.max(np.abs(complex_rpsi(rt) - complex_rpsi(rt_ref))) <= 1e-9
    run.g.close()


@pytest.mark.parametrize("method", METHODS)
@pytest.mark.parametrize("kind", ["ones", "zeros", "random"])
@pytest.mark.parametrize("thr", [-1.0, 0.0])
def test_methods_small_graphs(method, kind, thr):
    A, labels = kurgen.random_dense(700, 5, seed=61, p_in=0.85, p_out=0.03, symmetric=False)
    inst = kurgen.from_dense(A, labels, kind=kind, seed=5, K=2.5, h=0.02)
    _check(inst, method, dense_threshold=thr, tile_rows=128)


@pytest.mark.parametrize("method", METHODS)
def test_methods_complete_graph_cfg1(method):
    _check(kurgen.config(1), method, nsteps=20)


@pytest.mark.parametrize("method", METHODS)
def test_methods_cfg3(method):
    _check(kurgen.config(3), method, mode="matvec")


@pytest.mark.parametrize("method", METHODS)
def test_methods_with_remote_pass(method):
    """The separate k_remote pass (forced) under every integrator's stage epilogues."""
    inst = kurgen.sbm([2500, 1500, 900], np.array([[0.96, 0.004, 0.02], [0.004, 0.9, 0.003],
                                                    [0.02, 0.003, 0.25]]), 77, K=3.0, h=0.02)
    _check(inst, method, tile_rows=512, remote_pass=True, hot_min=1024)


@pytest.mark.parametrize("iters", [1, 2, 3])
def test_midpoint_iteration_cap(iters):
    """fp_max_iter caps the iterations exactly as the oracle does (tol 0 never converges early)."""
    inst = kurgen.sbm([900, 400], [[0.9, 0.02], [0.02, 0.7]], 13, K=3.0, h=0.05)
    _check(inst, "implicit_midpoint", fp_tol=0.0, fp_max_iter=iters)


def test_midpoint_residual_on_gpu():
    """The converged step solves theta_{n+1} = theta_n + h G((theta_n + theta_{n+1})/2)."""
    inst = kurgen.sbm([1500, 700], [[0.95, 0.01], [0.01, 0.5]], 17, K=4.0, h=0.01)
    run = Run(inst)
    th0 = run.theta_int.clone()
    th1 = th0.clone()
    kur.step_method(run.g, "implicit_midpoint", th1, run.omega_int, inst.K, inst.h, 1, fp_tol=1e-14, check=True)
    g = kur.rhs(run.g, (th0 + th1) / 2, run.omega_int, inst.K)
    res = (th1 - th0 - inst.h * g).abs().max().item()
    assert res <= 1e-13, res


def test_method_rk4_equals_kur_step():
    inst = kurgen.sbm([2000, 600], [[0.95, 0.01], [0.01, 0.4]], 3, K=2.0, h=0.01)
    run = Run(inst)
    a, b = run.theta_int.clone(), run.theta_int.clone()
    r1 = kur.step(run.g, a, run.omega_int, inst.K, inst.h, 5, 1)
    r2 = kur.step_method(run.g, "rk4", b, run.omega_int, inst.K, inst.h, 5, 1)
    assert torch.equal(a, b) and torch.equal(r1, r2)


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("method", METHODS)
def test_methods_group_bitwise(method, peer):
    """Sharded path (world 3, device-copy all-gather) bitwise equal to world 1 for every method."""
    inst = kurgen.sbm([3000, 500, 2000, 77], np.array(
        [[0.95, 0.01, 0.0, 0.6], [0.01, 0.3, 0.02, 0.0], [0.0, 0.02, 0.97, 0.1], [0.6, 0.0, 0.1, 0.5]]), 29,
        K=3.0, h=0.02)
    g1 = kur.graph_build(inst)
    th_full = g1.to_internal(torch.from_numpy(inst.theta0).cuda())
    om_full = g1.to_internal(torch.from_numpy(inst.omega).cuda())
    th1 = th_full.clone()
    rt1 = kur.step_method(g1, method, th1, om_full, inst.K, inst.h, 5, 1)
    gs = kur.group_build(inst, 3, peer_exchange=peer)
    ths = [th_full[g.row_begin:g.row_end].clone() for g in gs]
    oms = [om_full[g.row_begin:g.row_end].clone() for g in gs]
    rts = kur.group_step_method(gs, method, ths, oms, inst.K, inst.h, 5, 1)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat(ths), th1)
    for rt in rts:
        assert torch.equal(rt, rt1)


def test_method_errors():
    inst = kurgen.sbm([200], [[0.9]], 1)
    run = Run(inst)
    th = run.theta_int.clone()
    for kw in (dict(method="implicit_midpoint", fp_tol=-1.0), dict(method="implicit_midpoint", fp_max_iter=0)):
        with pytest.raises(kur.KurError) as e:
            kur.step_method(run.g, kw.pop("method"), th, run.omega_int, 1.0, 0.01, 1, **kw)
        assert e.value.status == 1
    with pytest.raises(kur.KurError) as e:
        kur._check(kur._lib.kur_step_method(run.g._h, 7, kur._dev_vec(th, run.g.n_local, 0, "t"),
                                             kur._dev_vec(run.omega_int, run.g.n_local, 0, "o"), 1.0, 0.01, 1, 0,
                                             None, 0.0, 1, kur._stream(None)))
    assert e.value.status == 1


def test_euler_nonfinite_flag():
    inst = kurgen.sbm([300], [[0.9]], 2)
    run = Run(inst)
    th = run.theta_int.clone()
    om = run.omega_int.clone()
    om[5] = float("inf")
    with pytest.raises(kur.KurError) as e:
        kur.step_method(run.g, "euler", th, om, 1.0, 0.01, 2, check=True)
    assert e.value.status == 9
