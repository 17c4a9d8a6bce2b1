"""GPU edge cases of the method against the oracle (the degenerate inputs the path must
handle): a single oscillator, two oscillators, a graph without edges, K = 0 and K < 0,
blocks at exactly the 50 % tie (reading R3: sparse), one-member communities, rows
without entries in an asymmetric graph, very large phases (the state is never wrapped,
R9), record_every beyond nsteps, and ragged tile tails."""
import math

import numpy as np
import pytest
import torch

import kurgen
import oracle
from paper_2102_07167_b200 import kur
from tests.helpers import R_TOL, Run, close, complex_rpsi

pytestmark = pytest.mark.gpu


def _both(inst, nsteps=5, mode="naive", **kw):
    run = Run(inst, **kw)
    f = run.rhs()
    f_ref = oracle.rhs(oracle.Graph(inst), inst.theta0, inst.omega, inst.K, mode=mode)
    th, rt = run.step(nsteps, 1)
    th_ref, _, rt_ref = oracle.rk4(oracle.Graph(inst), inst.theta0, inst.omega, inst.K, inst.h, nsteps, 1,
                                   mode=mode)
    return f, f_ref, th, th_ref, rt, rt_ref


def _check(inst, **kw):
    f, f_ref, th, th_ref, rt, rt_ref = _both(inst, **kw)
    ok, err = close(f, f_ref, abs_tol=1e-13, rel_tol=1e-12)
    assert ok, err
    ok, err = close(th, th_ref)
    assert ok, err
    assert np.max(np.abs(complex_rpsi(rt) - complex_rpsi(rt_ref))) <= R_TOL
    return f


def test_single_oscillator():
    inst = kurgen.from_dense(np.zeros((1, 1), np.uint8), [0], kind="ones", seed=1, K=3.0)
    f = _check(inst)
    assert f[0] == inst.omega[0]


def test_two_oscillators_both_encodings():
    A = np.array([[0, 1], [1, 0]], np.uint8)
    for kind in ("ones", "zeros"):
        _check(kurgen.from_dense(A, [0, 0], kind=kind, seed=2, K=1.5))


def test_graph_without_edges_gives_omega():
    n = 3000
    inst = kurgen.from_dense(np.zeros((n, n), np.uint8), np.arange(n) % 3, kind="ones", seed=3, K=2.0)
    f = _check(inst)
    assert np.array_equal(f, inst.omega)


@pytest.mark.parametrize("K", [0.0, -2.5])
def test_zero_and_repulsive_coupling(K):
    A, labels = kurgen.random_dense(900, 3, seed=5, p_in=0.9, p_out=0.05, symmetric=True)
    inst = kurgen.from_dense(A, labels, kind="auto", seed=5, K=K)
    f = _check(inst)
    if K == 0.0:
        assert np.array_equal(f, inst.omega)


def test_exact_tie_blocks():
    """A block with exactly as many zeros as ones (off-diagonal) is SPARSE (R3); result unchanged."""
    n = 64
    A = np.zeros((n, n), np.uint8)
    rng = np.random.default_rng(7)
    for i in range(n):  # each row of the single 64x64 block: 63 off-diagonal entries -> no exact tie per row,
        cols = [c for c in range(n) if c != i]  # so make the block-level census a tie
        A[i, rng.permutation(cols)[:(n - 1) // 2 + (i % 2)]] = 1
    ones = int(A.sum())
    zeros = n * (n - 1) - ones
    assert abs(ones - zeros) <= n  # near-tie census
    for thr in (-1.0, 0.5):
        _check(kurgen.from_dense(A, np.zeros(n, np.int32), kind="random", seed=8, K=2.0), dense_threshold=thr)


def test_singleton_communities_and_empty_rows():
    A, labels = kurgen.random_dense(500, 7, seed=9, p_in=0.8, p_out=0.1, symmetric=False)
    labels = labels.copy()
    labels[:5] = 7 + np.arange(5)  # five one-member communities
    A[10:20] = 0                   # rows without any edge (asymmetric A)
    _check(kurgen.from_dense(A, labels, kind="random", seed=9, K=2.0), tile_rows=64)


def test_large_phases_never_wrapped():
    """|theta| ~ 1e5: the state is not wrapped (R9); sincos of large arguments on both sides."""
    A, labels = kurgen.random_dense(700, 2, seed=11, p_in=0.9, p_out=0.1, symmetric=True)
    rng = np.random.default_rng(11)
    th0 = rng.uniform(-1e5, 1e5, 700)
    inst = kurgen.from_dense(A, labels, kind="auto", seed=11, K=2.0, theta0=th0)
    f, f_ref, th, th_ref, rt, rt_ref = _both(inst)
    assert close(f, f_ref, abs_tol=1e-11, rel_tol=1e-12)[0]
    assert close(th, th_ref, abs_tol=1e-9, rel_tol=1e-12)[0]
    assert np.max(np.abs(th)) > 9e4


def test_record_every_beyond_nsteps():
    inst = kurgen.sbm([400, 300], [[0.9, 0.05], [0.05, 0.8]], 13, K=2.0, h=0.02)
    run = Run(inst)
    th, rt = run.step(7, 10)
    assert rt.shape == (1, 2)
    r0 = oracle.order_parameter(inst.theta0)
    assert abs(rt[0, 0] - r0[0]) <= 1e-14


@pytest.mark.parametrize("n", [31, 32, 33, 511, 513, 2049, 4097])
def test_ragged_tile_tails(n):
    """Row counts around warp, chunk and tile boundaries (tiles of 512 rows, and the default)."""
    inst = kurgen.sbm([n // 2, n - n // 2], [[0.93, 0.03], [0.03, 0.6]], n, K=2.0)
    for kw in ({}, {"tile_rows": 512}):
        _check(inst, **kw)


@pytest.mark.parametrize("kind", ["ones", "zeros"])
def test_hot_chunk_lengths_every_remainder(kind):
    """Rows of 1..27 entries (non-zero or complement lists) inside one staged window:
    every remainder mod 9 of the 13-bit slot groups and both tail cases (plan.h)."""
    n = 27 * 32
    rng = np.random.default_rng(914)
    A = np.zeros((n, n), np.uint8) if kind == "ones" else np.ones((n, n), np.uint8)
    for j in range(n):
        cols = rng.choice(np.delete(np.arange(n), j), size=1 + (j % 27), replace=False)
        A[j, cols] = 1 if kind == "ones" else 0
    inst = kurgen.from_dense(A, np.zeros(n, np.int64), kind=kind, seed=5, K=3.0)
    _check(inst, hot_min=1)
