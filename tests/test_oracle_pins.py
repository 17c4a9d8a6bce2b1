"""Pins for the CPU oracle.

Each test ties oracle/ to something other than itself: a value hand-derived
from the paper's definition, a closed form, an identity of the paper, an
invariant, or a brute-force evaluation in higher precision.  All CPU-only.
"""
import json
import math
import os

import mpmath
import numpy as np
import pytest

import kurgen
import oracle
from oracle import bruteforce

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")
ENCODINGS = ("ones", "zeros", "auto", "random")


def _complete(n, theta, omega):
    A = np.ones((n, n), np.uint8) - np.eye(n, dtype=np.uint8)
    return kurgen.from_dense(A, np.zeros(n, np.int32), kind="zeros", theta0=theta, omega=omega)


# ---------------------------------------------------------------- O6 golden
def test_o6_spec_worked_examples():
    cases = json.load(open(GOLDEN))["cases"]
    for c in cases:
        th = np.array(c["theta"])
        if "expected_rhs" in c:
            inst = _complete(c["n"], th, np.array(c["omega"]))
            g = oracle.Graph(inst)
            for mode in ("naive", "matvec", "op"):
                f = oracle.rhs(g, th, inst.omega, c["K"], mode=mode)
                assert np.max(np.abs(f - np.array(c["expected_rhs"]))) <= c["tol_abs"], (c["name"], mode, f)
        if "expected_r" in c:
            r, psi = oracle.order_parameter(th)
            assert abs(r - c["expected_r"]) <= c["tol_abs"], (c["name"], r)
            if "expected_psi" in c:
                assert abs(psi - c["expected_psi"]) <= 1e-14


# ---------------------------------------------------------------- O1 mean-field identity
def test_o1_naive_equals_order_parameter_form_complete_graph():
    """(1/M) sum sin(theta_l - theta_m) = r sin(psi - theta_m)."""
    inst = kurgen.config(1)
    g = oracle.Graph(inst)
    th = inst.theta0.copy()
    for _ in range(3):  # theta(0) and two further states along the flow
        fn = oracle.rhs(g, th, inst.omega, inst.K, mode="naive")
        fo = oracle.rhs(g, th, inst.omega, inst.K, mode="op")
        assert np.max(np.abs(fn - fo)) <= 1e-13
        th = th + 0.05 * fn


# ---------------------------------------------------------------- O2 brute force
@pytest.mark.parametrize("n", [2, 3, 8, 64])
@pytest.mark.parametrize("kind", ENCODINGS)
def test_o2_bruteforce_tiny(n, kind):
    C = 1 if n < 8 else 3
    A, labels = kurgen.random_dense(n, C, seed=100 + n, p_in=0.7, p_out=0.3, symmetric=False)
    inst = kurgen.from_dense(A, labels, kind=kind, seed=n)
    g = oracle.Graph(inst)
    K = 1.7
    ref = bruteforce.rhs_fsum(A, inst.theta0, inst.omega, K)
    mp = bruteforce.rhs_mp(A, inst.theta0, inst.omega, K)
    mpf = np.array([float(x) for x in mp])
    ulp = np.spacing(np.maximum(np.abs(ref), 1.0))
    for mode in ("naive", "matvec"):
        f = oracle.rhs(g, inst.theta0, inst.omega, K, mode=mode)
        assert np.all(np.abs(f - ref) <= 4 * n * ulp + 1e-15), (mode, np.max(np.abs(f - ref)))
        assert np.all(np.abs(f - mpf) <= 4 * n * ulp + 1e-15), (mode, np.max(np.abs(f - mpf)))


def test_o2_encodings_are_bitwise_identical():
    """KUR_ONES / KUR_ZEROS decodings enumerate the same ones in the same order."""
    A, labels = kurgen.random_dense(120, 5, seed=3, p_in=0.85, p_out=0.05, symmetric=True)
    outs = []
    for kind in ENCODINGS:
        inst = kurgen.from_dense(A, labels, kind=kind, seed=1)
        g = oracle.Graph(inst)
        outs.append(oracle.rhs(g, inst.theta0, inst.omega, 2.0, mode="naive"))
        assert np.array_equal(g.degree(), A.sum(1) - np.diag(A))
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_order_parameter_mp():
    th = kurgen.uniform(5, 2, 64, 0.0, 2 * math.pi)
    r, psi = oracle.order_parameter(th)
    z = bruteforce.order_parameter_mp(th)
    assert abs(r - float(abs(z))) <= 1e-15
    assert abs(r * math.cos(psi) - float(z.real)) <= 1e-15
    assert abs(r * math.sin(psi) - float(z.imag)) <= 1e-15


# ---------------------------------------------------------------- O3 conservation
@pytest.mark.parametrize("which", ["cfg1", "cfg3", "sbm"])
def test_o3_conserved_mean_phase_velocity(which):
    """Symmetric A, uniform scaling: sum_m (f_m - omega_m) = 0."""
    if which == "cfg1":
        inst = kurgen.config(1)
    elif which == "cfg3":
        inst = kurgen.config(3)
    else:
        inst = kurgen.sbm([300, 200, 77, 1], [[0.9, 0.01, 0.6, 0.1], [0.01, 0.3, 0.0, 0.0],
                                              [0.6, 0.0, 0.97, 0.5], [0.1, 0.0, 0.5, 0.0]], 11)
    g = oracle.Graph(inst)
    for mode in ("naive", "matvec"):
        f = oracle.rhs(g, inst.theta0, inst.omega, inst.K, mode=mode)
        d = f - inst.omega
        assert abs(math.fsum(d)) <= 1e-12 * np.sum(np.abs(d)) + 1e-13, mode


def test_o3_conservation_fails_for_asymmetric():
    """Non-vacuity: an asymmetric A breaks the identity."""
    A, labels = kurgen.random_dense(64, 2, seed=9, p_in=0.6, p_out=0.2, symmetric=False)
    inst = kurgen.from_dense(A, labels, seed=4)
    g = oracle.Graph(inst)
    d = oracle.rhs(g, inst.theta0, inst.omega, 3.0) - inst.omega
    assert abs(math.fsum(d)) > 1e-6


def test_o3_conservation_along_rk4():
    """RK4 preserves linear invariants: sum theta(t_n) - sum theta(0) - t_n sum omega ~ 0."""
    inst = kurgen.sbm([100, 150, 50], [[0.9, 0.02, 0.0], [0.02, 0.7, 0.3], [0.0, 0.3, 0.1]], 21,
                      K=4.0, h=0.01, nsteps=40)
    g = oracle.Graph(inst)
    for nst in (10, 40):
        th, _, _ = oracle.rk4(g, inst.theta0, inst.omega, inst.K, inst.h, nst, 0, mode="naive")
        res = math.fsum(th) - math.fsum(inst.theta0) - nst * inst.h * math.fsum(inst.omega)
        assert abs(res) <= 1e-10 * inst.n


# ---------------------------------------------------------------- O4 synchronisation
@pytest.mark.parametrize("n,mode", [(1000, "op"), (120, "naive"), (120, "matvec")])
def test_o4_synchronisation_identical_frequencies(n, mode):
    """omega = 0, K > 0: gradient flow of V = (KM/2)(1 - r^2) => r nondecreasing -> 1."""
    th0 = kurgen.uniform(77, 2, n, 0.0, 2 * math.pi)
    inst = _complete(n, th0, np.zeros(n))
    g = oracle.Graph(inst)
    _, _, rt = oracle.rk4(g, th0, inst.omega, 2.0, 0.01, 3000, 1, mode=mode)
    r = rt[:, 0]
    assert np.all(np.diff(r) >= -1e-12)
    assert r[-1] >= 1 - 1e-10


# ---------------------------------------------------------------- O5 RK4 order
def _adler_exact(t, K, w, th1_0, th2_0):
    """Two identical oscillators (complete graph, M=2): phi=th2-th1 obeys phi'=-K sin(phi),
    tan(phi/2) = tan(phi0/2) e^{-Kt}; th1+th2 = const + 2 w t."""
    phi0 = th2_0 - th1_0
    phi = 2.0 * math.atan(math.tan(phi0 / 2.0) * math.exp(-K * t))
    s = th1_0 + th2_0 + 2.0 * w * t
    return (s - phi) / 2.0, (s + phi) / 2.0


@pytest.mark.parametrize("mode", ["naive", "matvec", "op"])
def test_o5_rk4_order_four(mode):
    K, w, T = 1.0, 0.3, 2.0
    th0 = np.array([0.1, 2.1])
    inst = _complete(2, th0, np.array([w, w]))
    g = oracle.Graph(inst)
    ex = np.array(_adler_exact(T, K, w, *th0))
    errs = []
    for h in (0.2, 0.1, 0.05, 0.025):
        th, _, _ = oracle.rk4(g, th0, inst.omega, K, h, int(round(T / h)), 0, mode=mode)
        errs.append(np.max(np.abs(th - ex)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert all(3.8 <= o <= 4.2 for o in orders), orders


def test_o5_rk4_self_convergence_n64():
    inst = kurgen.sbm([40, 24], [[0.8, 0.1], [0.1, 0.9]], 5, K=3.0)
    g = oracle.Graph(inst)
    T = 1.0
    ref, _, _ = oracle.rk4(g, inst.theta0, inst.omega, inst.K, T / 1024, 1024, 0, mode="matvec")
    errs = []
    for nst in (8, 16, 32):
        th, _, _ = oracle.rk4(g, inst.theta0, inst.omega, inst.K, T / nst, nst, 0, mode="matvec")
        errs.append(np.max(np.abs(th - ref)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert all(3.7 <= o <= 4.3 for o in orders), orders


# ---------------------------------------------------------------- O7 splay state
def test_o7_splay_state_incoherent():
    """theta_m = 2 pi m / M: roots of unity sum to zero => r = 0 and f = omega."""
    n = 1000
    th = 2 * math.pi * np.arange(1, n + 1) / n
    inst = _complete(n, th, kurgen.normal(1, 1, n))
    g = oracle.Graph(inst)
    r, _ = oracle.order_parameter(th)
    assert r <= 1e-13
    for mode in ("naive", "matvec", "op"):
        f = oracle.rhs(g, th, inst.omega, 3.0, mode=mode)
        assert np.max(np.abs(f - inst.omega)) <= 1e-12


# ---------------------------------------------------------------- O8 invariances
def test_o8_global_shift_invariance():
    A, labels = kurgen.random_dense(200, 4, seed=8, p_in=0.8, p_out=0.05)
    inst = kurgen.from_dense(A, labels, seed=2)
    g = oracle.Graph(inst)
    f0 = oracle.rhs(g, inst.theta0, inst.omega, 2.0)
    f1 = oracle.rhs(g, inst.theta0 + 1.2345, inst.omega, 2.0)
    assert np.max(np.abs(f1 - f0)) <= 1e-13
    r0, p0 = oracle.order_parameter(inst.theta0)
    r1, p1 = oracle.order_parameter(inst.theta0 + 1.2345)
    assert abs(r1 - r0) <= 1e-14
    assert abs(math.remainder(p1 - p0 - 1.2345, 2 * math.pi)) <= 1e-13


def test_o8_relabelling_equivariance():
    """permute A, theta, omega by P  =>  RHS permuted by P."""
    A, labels = kurgen.random_dense(150, 3, seed=12, p_in=0.75, p_out=0.1, symmetric=False)
    inst = kurgen.from_dense(A, labels, seed=3)
    perm = kurgen.permutation(44, 6, 150)  # new position i holds old node perm[i]
    Ap = A[np.ix_(perm, perm)]
    instp = kurgen.from_dense(Ap, labels[perm], kind="random", seed=5,
                              theta0=inst.theta0[perm], omega=inst.omega[perm])
    f = oracle.rhs(oracle.Graph(inst), inst.theta0, inst.omega, 2.5)
    fp = oracle.rhs(oracle.Graph(instp), instp.theta0, instp.omega, 2.5)
    assert np.max(np.abs(fp - f[perm])) <= 1e-13


# ---------------------------------------------------------------- O9 naive == matvec
@pytest.mark.parametrize("which", ["cfg1", "cfg3", "sbm", "cfg4_rows", "cfg5_rows"])
def test_o9_naive_equals_matvec(which):
    """O9: the P:388 definition (per-edge sines) and the P:443 componentwise form agree,
    on whole configs 1 and 3 and on sampled rows (1024 + a whole community) of the full configs 4 and 5."""
    rows = None
    if which == "cfg1":
        inst = kurgen.config(1)
    elif which == "cfg3":
        inst = kurgen.config(3)
    elif which in ("cfg4_rows", "cfg5_rows"):
        c = 4 if which == "cfg4_rows" else 5
        inst = kurgen.config(c)
        rnd = (kurgen.raw_bits(c, 11, 1024) % np.uint64(inst.n)).astype(np.int64)
        rows = np.concatenate([rnd, np.flatnonzero(inst.community == 1)[:2048].astype(np.int64)])
    else:
        inst = kurgen.sbm([500, 300, 10], [[0.95, 0.2, 0.6], [0.2, 0.05, 0.0], [0.6, 0.0, 1.0]], 31)
    g = oracle.Graph(inst)
    fn = oracle.rhs(g, inst.theta0, inst.omega, inst.K, mode="naive", rows=rows)
    fm = oracle.rhs(g, inst.theta0, inst.omega, inst.K, mode="matvec", rows=rows)
    om = inst.omega if rows is None else inst.omega[rows]
    scale = np.abs(fn - om) + np.abs(om)
    assert np.all(np.abs(fn - fm) <= 1e-12 * scale + 1e-13)
    assert np.median(np.abs(fn - om)) > 1e-6  # the coupling term is not vacuous on these rows


def test_sampled_rows_match_full():
    inst = kurgen.config(3)
    g = oracle.Graph(inst)
    rows = np.array([0, 17, 4095, 65535, 30000], np.int64)
    full = oracle.rhs(g, inst.theta0, inst.omega, inst.K, mode="naive")
    part = oracle.rhs(g, inst.theta0, inst.omega, inst.K, mode="naive", rows=rows)
    assert np.array_equal(part, full[rows])


def test_thread_count_invariance():
    inst = kurgen.sbm([200, 100], [[0.9, 0.05], [0.05, 0.5]], 41)
    g = oracle.Graph(inst)
    t0 = oracle.num_threads()
    try:
        oracle.set_num_threads(1)
        a = oracle.rhs(g, inst.theta0, inst.omega, 2.0, mode="naive")
        oracle.set_num_threads(max(2, t0))
        b = oracle.rhs(g, inst.theta0, inst.omega, 2.0, mode="naive")
    finally:
        oracle.set_num_threads(t0)
    assert np.array_equal(a, b)


# ---------------------------------------------------------------- r(t) recording schedule (R10)
def _adler_rpsi(t, K, w, th0):
    """r e^{i psi} = (e^{i th1} + e^{i th2}) / 2 of the closed-form two-oscillator solution."""
    a, b = _adler_exact(t, K, w, *th0)
    return (complex(math.cos(a), math.sin(a)) + complex(math.cos(b), math.sin(b))) / 2.0


@pytest.mark.parametrize("mode", ["naive", "matvec", "op"])
def test_rk4_records_r_on_schedule_adler(mode):
    """orc_rk4 records r e^{i psi} of theta_n at n = 0, k, 2k, ... (reading R10, before stepping) and
    captures theta after 10 steps: both against the Adler closed form at t = n h (RK4 error ~1e-11 at
    h = 0.01); a schedule shifted by one step would be off by ~|dr/dt| h ~ 4e-3."""
    K, w, h, k, nsteps = 1.0, 0.3, 0.01, 5, 200
    th0 = np.array([0.1, 2.1])
    inst = _complete(2, th0, np.array([w, w]))
    g = oracle.Graph(inst)
    _, th10, rt = oracle.rk4(g, th0, inst.omega, K, h, nsteps, k, mode=mode)
    assert rt.shape == (nsteps // k + 1, 2)
    got = rt[:, 0] * np.exp(1j * rt[:, 1])
    t = np.arange(rt.shape[0]) * k * h
    exact = np.array([_adler_rpsi(ti, K, w, th0) for ti in t])
    assert np.max(np.abs(got - exact)) <= 1e-9
    shifted = np.array([_adler_rpsi(ti + h, K, w, th0) for ti in t])
    assert np.max(np.abs(got - shifted)) > 1e-4  # non-vacuity of the bound above
    assert np.max(np.abs(th10 - np.array(_adler_exact(10 * h, K, w, *th0)))) <= 1e-11
    # a trajectory shorter than 10 steps: theta10 is not captured past nsteps, the final state is
    th, _, rt3 = oracle.rk4(g, th0, inst.omega, K, h, 3, 1, mode=mode)
    assert rt3.shape == (4, 2)
    assert np.max(np.abs(th - np.array(_adler_exact(3 * h, K, w, *th0)))) <= 1e-12


@pytest.mark.parametrize("method,order", [("euler", 1), ("heun", 2), ("implicit_midpoint", 2)])
def test_step_method_records_r_on_schedule(method, order):
    """orc_step_method's r(t) samples: rt[i] is the order parameter of theta after i*k steps (the
    same method run for exactly i*k steps, then the plain definition), and for the
    second-order methods within C h^2 of the Adler closed form (a one-step shift costs ~4e-3)."""
    K, w, h, k, nsteps = 1.0, 0.3, 0.01, 4, 100
    th0 = np.array([0.1, 2.1])
    inst = _complete(2, th0, np.array([w, w]))
    g = oracle.Graph(inst)
    _, rt = oracle.step_method(g, method, th0, inst.omega, K, h, nsteps, k)
    assert rt.shape == (nsteps // k + 1, 2)
    for i in (0, 1, 7, nsteps // k):
        thi, _ = oracle.step_method(g, method, th0, inst.omega, K, h, i * k, 0)
        z = np.exp(1j * thi).mean()
        assert abs(rt[i, 0] * np.exp(1j * rt[i, 1]) - z) <= 1e-15, (method, i)
    got = rt[:, 0] * np.exp(1j * rt[:, 1])
    t = np.arange(rt.shape[0]) * k * h
    exact = np.array([_adler_rpsi(ti, K, w, th0) for ti in t])
    err = np.max(np.abs(got - exact))
    assert err <= (5e-4 if order == 2 else 1e-2), err
