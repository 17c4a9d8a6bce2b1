"""GPU parity of the cluster-resident stage (k_stage_cz: world 1, n <= 65536, all of z
staged over one 8-CTA cluster, row sums added through distributed shared memory) against the CPU
oracle, for every integrator and the potential, plus its agreement with the tile plan (another
summation order: within rounding, not bitwise)."""
import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import Run, close, complex_rpsi

pytestmark = pytest.mark.gpu


def _inst(scaling=0):
    """Dense and sparse diagonal blocks, a dense off-diagonal pair, a 7-node and an empty-ish community,
    permuted labels; n = 15207 (4 windows), so the cluster plan takes it."""
    P = np.array([[0.95, 0.002, 0.9, 0.0, 0.0, 0.001],
                  [0.002, 0.3, 0.0, 0.0, 0.0, 0.0],
                  [0.9, 0.0, 0.97, 0.001, 0.0, 0.0],
                  [0.0, 0.0, 0.001, 0.05, 0.0, 0.0],
                  [0.0, 0.0, 0.0, 0.0, 0.5, 0.0],
                  [0.001, 0.0, 0.0, 0.0, 0.0, 0.6]])
    inst = kurgen.sbm([5000, 3000, 4000, 1200, 7, 2000], P, 20210215, K=2.0, h=0.01)
    inst.scaling = scaling
    return inst


def test_cluster_plan_is_chosen():
    for inst in (_inst(), kurgen.config(3)):
        run = Run(inst)
        assert run.g.info["cluster_plan"] > 0, run.g.info
        assert Run(inst, tile_mode=True).g.info["cluster_plan"] == 0
    assert Run(kurgen.config(4)).g.info["cluster_plan"] == 0  # n = 262144 > 65536


@pytest.mark.parametrize("scaling", [0, 1])
def test_cluster_rhs_and_rk4_vs_oracle(scaling):
    inst = _inst(scaling)
    og = oracle.Graph(inst)
    run = Run(inst)
    ok, err = close(run.rhs(), oracle.rhs(og, inst.theta0, inst.omega, inst.K, mode="naive"), abs_tol=1e-13)
    assert ok, err
    _, th10_ref, rt_ref = oracle.rk4(og, inst.theta0, inst.omega, inst.K, inst.h, 10, 1, mode="naive")
    th10, rt = run.step(10, 1)
    ok, err = close(th10, th10_ref)
    assert ok, err
    assert np.max(np.abs(complex_rpsi(rt) - complex_rpsi(rt_ref))) <= 1e-9


@pytest.mark.parametrize("method", ["euler", "heun", "implicit_midpoint"])
def test_cluster_methods_vs_oracle(method):
    inst = _inst()
    run = Run(inst)
    th = run.theta_int.clone()
    rt = kur.step_method(run.g, method, th, run.omega_int, inst.K, inst.h, 8, 2, check=True)
    th_ref, rt_ref = oracle.step_method(oracle.Graph(inst), method, inst.theta0, inst.omega, inst.K, inst.h, 8, 2,
                                        mode="naive")
    ok, err = close(run.user(th), th_ref)
    assert ok, (method, err)
    assert np.max(np.abs(complex_rpsi(rt.cpu().numpy()) - complex_rpsi(rt_ref))) <= 1e-9


def test_cluster_potential_vs_oracle():
    inst = _inst()
    run = Run(inst)
    got = float(kur.potential(run.g, run.theta_int, run.omega_int, inst.K).item())
    ref = oracle.potential(oracle.Graph(inst), inst.theta0, inst.omega, inst.K)
    assert abs(got - ref) <= 1e-11 * (1 + abs(ref)), (got, ref)


def test_cluster_vs_tile_plan_and_determinism():
    """Same trajectory as the tile plan up to rounding (different summation order), and bitwise
    reproducible run to run (no atomics: fixed part order, fixed DSMEM rank order)."""
    inst = kurgen.config(3)
    a, b, t = Run(inst), Run(inst), Run(inst, tile_mode=True)
    fa, fb, ft = a.rhs(), b.rhs(), t.rhs()
    assert np.array_equal(fa, fb)
    ok, err = close(fa, ft, abs_tol=1e-13, rel_tol=1e-13)
    assert ok, err
    tha, rta = a.step(20, 5)
    thb, rtb = b.step(20, 5)
    tht, rtt = t.step(20, 5)
    assert np.array_equal(tha, thb) and np.array_equal(rta, rtb)
    ok, err = close(tha, tht, abs_tol=1e-11, rel_tol=1e-12)
    assert ok, err


def test_cluster_nonfinite_flag():
    inst = _inst()
    inst.omega = inst.omega.copy()
    inst.omega[123] = np.inf
    run = Run(inst)
    th = run.theta_int.clone()
    with pytest.raises(kur.KurError) as e:
        kur.step(run.g, th, run.omega_int, inst.K, inst.h, 2, 0, check=True)
    assert e.value.status == 9
