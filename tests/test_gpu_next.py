"""GPU parity for the NEXT rows: non-uniform (degree) scaling and the
potential V through kur_potential, against the CPU oracle."""
import math

import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import Run, close, complex_rpsi

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("remote_pass", [None, True])
@pytest.mark.parametrize("kind", ["ones", "zeros", "random"])
@pytest.mark.parametrize("thr", [-1.0, 0.0, 1.0])
def test_degree_scaling_small(kind, thr, remote_pass):
    A, labels = kurgen.random_dense(400, 4, seed=44, p_in=0.8, p_out=0.05, symmetric=False)
    np.fill_diagonal(A[:50, :50], 1)  # some stored self-loops (count in the degree, R22)
    A[3] = 0  # zero row (no self-loop either) -> theta' = omega exactly
    inst = kurgen.from_dense(A, labels, kind=kind, seed=9, K=2.0, scaling=1, self_loops=True)
    ref = oracle.rhs(oracle.Graph(inst), inst.theta0, inst.omega, inst.K, mode="naive")
    got = Run(inst, dense_threshold=thr, remote_pass=remote_pass, tile_rows=128).rhs()
    ok, err = close(got, ref, abs_tol=1e-13, rel_tol=1e-12)
    assert ok, err
    i3 = int(np.flatnonzero(np.arange(400) == 3)[0])
    assert got[i3] == inst.omega[i3]


def test_degree_scaling_cfg3_trajectory():
    inst = kurgen.config(3)
    inst.scaling = 1
    og = oracle.Graph(inst)
    run = Run(inst)
    f_ref = oracle.rhs(og, inst.theta0, inst.omega, inst.K, mode="matvec")
    assert close(run.rhs(), f_ref)[0]
    _, th10_ref, rt_ref = oracle.rk4(og, inst.theta0, inst.omega, inst.K, inst.h, 10, 1, mode="matvec")
    th10, rt = run.step(10, 1)
    ok, err = close(th10, th10_ref)
    assert ok, err
    assert np.max(np.abs(complex_rpsi(rt) - complex_rpsi(rt_ref))) <= 1e-9


def _gpu_potential(inst, **kw):
    run = Run(inst, **kw)
    return float(kur.potential(run.g, run.theta_int, run.omega_int, inst.K).item())


@pytest.mark.parametrize("scaling", [0, 1])
def test_potential_small(scaling):
    for seed, (n, C, sym) in enumerate([(60, 1, True), (300, 3, False), (1200, 5, True)]):
        A, labels = kurgen.random_dense(n, C, seed=seed + 70, p_in=0.85, p_out=0.04, symmetric=sym)
        inst = kurgen.from_dense(A, labels, kind="random", seed=seed, K=1.3, scaling=scaling)
        ref = oracle.potential(oracle.Graph(inst), inst.theta0, inst.omega, inst.K)
        for thr in (-1.0, 0.0):
            got = _gpu_potential(inst, dense_threshold=thr)
            assert abs(got - ref) <= 1e-11 * (1 + abs(ref)), (n, scaling, thr, got, ref)


def test_potential_configs_1_and_3():
    for k in (1, 3):
        inst = kurgen.config(k)
        ref = oracle.potential(oracle.Graph(inst), inst.theta0, inst.omega, inst.K)
        got = _gpu_potential(inst)
        assert abs(got - ref) <= 1e-11 * (1 + abs(ref)), (k, got, ref)


def test_potential_decreases_on_gpu():
    """P:212-218 on the device path: V(theta_{n+1}) <= V(theta_n) along kur_step (symmetric, uniform)."""
    inst = kurgen.sbm([3000, 1000], [[0.95, 0.01], [0.01, 0.6]], 8, K=4.0, h=0.01)
    run = Run(inst)
    th = run.theta_int.clone()
    v = float(kur.potential(run.g, th, run.omega_int, inst.K).item())
    for _ in range(10):
        kur.step(run.g, th, run.omega_int, inst.K, inst.h, 1)
        v2 = float(kur.potential(run.g, th, run.omega_int, inst.K).item())
        assert v2 <= v + 1e-9 * abs(v)
        v = v2
