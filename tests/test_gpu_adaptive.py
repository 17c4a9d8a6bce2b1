"""GPU parity for NEXT-4's variable-step RK4 (reading R25): kur_integrate_adaptive
against oracle.integrate_adaptive on the same seeded inputs.  The controller decides on
the error estimate in fp64 on both sides, so the accepted step sequences agree (the
estimates differ only by summation order); times and h to 1e-12, theta(t_end) and the
complex order parameter at every accepted step within north_star's tolerances."""
import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import R_TOL, Run, close, complex_rpsi

pytestmark = pytest.mark.gpu


def _both(inst, t_end, h0, mode="naive", **ctrl):
    run = Run(inst, **{k: ctrl.pop(k) for k in list(ctrl) if k in ("remote_pass", "tile_rows")})
    th = run.theta_int.clone()
    t, h, rp, rej = kur.integrate_adaptive(run.g, th, run.omega_int, inst.K, t_end, h0, **ctrl)
    torch.cuda.synchronize()
    ref = oracle.integrate_adaptive(oracle.Graph(inst), inst.theta0, inst.omega, inst.K, t_end, h0, mode=mode,
                                    **ctrl)
    return run, run.user(th), t, h, rp, rej, ref


@pytest.mark.parametrize("tol", [1e-6, 1e-10])
def test_adaptive_small_sbm(tol):
    inst = kurgen.sbm([1200, 800, 300], np.array([[0.95, 0.01, 0.3], [0.01, 0.9, 0.0], [0.3, 0.0, 0.6]]), 41,
                      K=4.0)
    run, th, t, h, rp, rej, (th_r, t_r, h_r, rp_r, rej_r) = _both(inst, 0.5, 0.05, atol=tol, rtol=tol)
    assert len(t) == len(t_r) and rej == rej_r, (len(t), len(t_r), rej, rej_r)
    assert np.max(np.abs(t - t_r)) <= 1e-6 * 0.5 and np.max(np.abs(h / h_r - 1)) <= 1e-6
    assert t[-1] == 0.5
    ok, err = close(th, th_r)
    assert ok, err
    assert np.max(np.abs(complex_rpsi(rp) - complex_rpsi(rp_r))) <= R_TOL


def test_adaptive_cfg3_remote_pass():
    inst = kurgen.config(3)
    run, th, t, h, rp, rej, (th_r, t_r, h_r, rp_r, rej_r) = _both(inst, 0.05, 0.02, mode="matvec", atol=1e-8,
                                                                  rtol=1e-8, remote_pass=True)
    assert len(t) == len(t_r) and rej == rej_r
    ok, err = close(th, th_r)
    assert ok, err


def test_adaptive_loose_equals_fixed_step_on_gpu():
    """Every trial accepted at h_max: the device result equals kur_step with h_max/2 bitwise."""
    inst = kurgen.sbm([2000, 500], [[0.95, 0.02], [0.02, 0.5]], 8, K=2.0)
    run = Run(inst)
    a = run.theta_int.clone()
    t, h, rp, rej = kur.integrate_adaptive(run.g, a, run.omega_int, inst.K, 0.5, 0.0625, atol=1e6, rtol=0.0,
                                           h_max=0.0625)
    b = run.theta_int.clone()
    kur.step(run.g, b, run.omega_int, inst.K, 0.03125, 16)
    torch.cuda.synchronize()
    assert rej == 0 and len(t) == 8 and torch.equal(a, b)


def test_adaptive_errors():
    inst = kurgen.sbm([300], [[0.9]], 3)
    run = Run(inst)
    th = run.theta_int.clone()
    with pytest.raises(kur.KurError) as e:
        kur.integrate_adaptive(run.g, th, run.omega_int, 1.0, -1.0, 0.1)
    assert e.value.status == 1
    with pytest.raises(kur.KurError) as e:  # impossible tolerance with a large h_min
        kur.integrate_adaptive(run.g, th, run.omega_int, 50.0, 1.0, 0.5, atol=1e-15, rtol=0.0, h_min=0.25)
    assert e.value.status == 11


@pytest.mark.parametrize("peer", [False, True])
def test_adaptive_group_bitwise(peer):
    """Sharded variable-step RK4 (world 3): the same accepted steps and bitwise the same state as world 1."""
    inst = kurgen.sbm([3000, 500, 2000, 77], np.array(
        [[0.95, 0.01, 0.0, 0.6], [0.01, 0.3, 0.02, 0.0], [0.0, 0.02, 0.97, 0.1], [0.6, 0.0, 0.1, 0.5]]), 29,
        K=3.0)
    g1 = kur.graph_build(inst)
    full = g1.to_internal(torch.from_numpy(inst.theta0).cuda())
    omf = g1.to_internal(torch.from_numpy(inst.omega).cuda())
    th1 = full.clone()
    t1, h1, rp1, rej1 = kur.integrate_adaptive(g1, th1, omf, inst.K, 0.3, 0.05, atol=1e-8, rtol=1e-8)
    gs = kur.group_build(inst, 3, peer_exchange=peer)
    ths = [full[g.row_begin:g.row_end].clone() for g in gs]
    oms = [omf[g.row_begin:g.row_end].clone() for g in gs]
    t3, h3, rp3, rej3 = kur.group_integrate_adaptive(gs, ths, oms, inst.K, 0.3, 0.05, atol=1e-8, rtol=1e-8)
    torch.cuda.synchronize()
    assert rej3 == rej1 and np.array_equal(t3, t1) and np.array_equal(h3, h1) and np.array_equal(rp3, rp1)
    assert torch.equal(torch.cat(ths), th1)


def _paper_fig2_instance(M, K):
    """omega_m = 1 + omega_0 (2m - M - 1)/(M - 1) with omega_0 = 2,
    theta_m(0) = 2 pi m / M, complete graph (the classical model), coupling K."""
    m = np.arange(1, M + 1)
    A = np.ones((M, M), np.uint8) - np.eye(M, dtype=np.uint8)
    return kurgen.from_dense(A, np.zeros(M, np.int64), kind="zeros", omega=1.0 + 2.0 * (2 * m - M - 1) / (M - 1),
                             theta0=2 * np.pi * m / M, K=K)


@pytest.mark.parametrize("K", [1.0, 5.0])
def test_paper_synchronisation_claim_k5(K):
    """P:361-375 (Figs. 2-5): M = 10^2, T = 200, variable-step RK4: "the modulus of the complex order
    parameter is close to one for K = 5" (qualitative, not a parity number the paper prints); K = 1 stays
    far from synchrony.  GPU and oracle take the same accepted steps and agree on r e^{i psi}."""
    inst = _paper_fig2_instance(100, K)
    run, th, t, h, rp, rej, (th_r, t_r, h_r, rp_r, rej_r) = _both(inst, 200.0, 0.01, mode="naive", atol=1e-8,
                                                                  rtol=1e-8)
    assert len(t) == len(t_r) and rej == rej_r and t[-1] == 200.0
    assert np.max(np.abs(complex_rpsi(rp) - complex_rpsi(rp_r))) <= R_TOL
    r_end = rp[-1, 0]
    if K == 5.0:
        assert r_end >= 0.9, r_end
        assert np.all(rp[len(rp) // 2:, 0] >= 0.9)  # locked for the second half of [0, T]
    else:
        assert r_end <= 0.5, r_end
