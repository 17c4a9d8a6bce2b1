"""oracle — plain, slow, obviously correct CPU reference for the hot path.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product (``paper_2102_07167_b200``) never imports it and shares
no code with it (see ``kur_oracle.c``'s header for what it computes and the
PAPER.md passages each function follows).

Pins (what ties the oracle to the paper rather than to itself) live in
``tests/test_oracle_pins.py``; see DESIGN.md §3 for the list.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_LIB = os.path.join(_HERE, "liboracle.so")

NAIVE, MATVEC, OP = 0, 1, 2
_MODES = {"naive": NAIVE, "matvec": MATVEC, "op": OP}


def _load():
    if not os.path.exists(_LIB):
        subprocess.run(["make", "-s", "-C", _ROOT, "oracle/liboracle.so"], check=True)
    lib = ctypes.CDLL(_LIB)
    p, i64, i32, d = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    lib.orc_graph_new.argtypes = [i64, i32, p, p, p, p, p, p]
    lib.orc_graph_new.restype = p
    lib.orc_graph_free.argtypes = [p]
    lib.orc_rhs.argtypes = [p, ctypes.c_int, d, p, p, i64, p, p]
    lib.orc_rhs.restype = ctypes.c_int
    lib.orc_rk4.argtypes = [p, ctypes.c_int, d, d, i64, i32, p, p, p, p]
    lib.orc_rk4.restype = ctypes.c_int
    lib.orc_order_parameter.argtypes = [i64, p, p]
    lib.orc_row_degree.argtypes = [p, p]
    lib.orc_num_threads.restype = ctypes.c_int
    lib.orc_graph_set_scaling.argtypes = [p, ctypes.c_int]
    lib.orc_potential.argtypes = [p, d, p, p]
    lib.orc_potential.restype = d
    lib.orc_set_num_threads.argtypes = [ctypes.c_int]
    lib.orc_step_method.argtypes = [p, ctypes.c_int, ctypes.c_int, d, d, i64, i32, p, p, p, d, i32]
    lib.orc_step_method.restype = ctypes.c_int
    lib.orc_integrate_adaptive.argtypes = [p, ctypes.c_int, d, d, d, d, d, d, d, d, d, d, i64, p, p, i64, p, p, p,
                                           p]
    lib.orc_integrate_adaptive.restype = i64
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def num_threads():
    return lib().orc_num_threads()


def set_num_threads(t):
    lib().orc_set_num_threads(int(t))


class Graph:
    """Holds the caller's arrays (kept alive here) plus community member lists."""

    def __init__(self, inst):
        self._keep = [np.ascontiguousarray(a) for a in (
            inst.community.astype(np.int32, copy=False), inst.seg_ptr.astype(np.int64, copy=False),
            inst.seg_comm.astype(np.int32, copy=False), inst.seg_kind.astype(np.uint8, copy=False),
            inst.idx_ptr.astype(np.int64, copy=False), inst.idx.astype(np.int32, copy=False))]
        self.n = int(inst.n)
        self._h = lib().orc_graph_new(self.n, int(inst.n_comm), *[_p(a) for a in self._keep])
        self.scaling = int(getattr(inst, "scaling", 0))
        lib().orc_graph_set_scaling(self._h, self.scaling)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_graph_free(self._h)
            self._h = None

    def degree(self):
        out = np.empty(self.n, np.int64)
        lib().orc_row_degree(self._h, _p(out))
        return out


def rhs(g: Graph, theta, omega, K, mode="naive", rows=None):
    """Right-hand side (user order).  rows: optional int64 user ids to evaluate."""
    theta = np.ascontiguousarray(theta, np.float64)
    omega = np.ascontiguousarray(omega, np.float64)
    if rows is not None:
        rows = np.ascontiguousarray(rows, np.int64)
        out = np.empty(rows.shape[0], np.float64)
        nr = rows.shape[0]
    else:
        out = np.empty(g.n, np.float64)
        nr = 0
    rc = lib().orc_rhs(g._h, _MODES[mode], float(K), _p(theta), _p(omega), nr, _p(rows), _p(out))
    if rc:
        raise ValueError("orc_rhs failed")
    return out


def rk4(g: Graph, theta0, omega, K, h, nsteps, record_every=1, mode="matvec"):
    """Classical RK4; returns (theta_final, theta_after_10_steps, r_trace[nrec, 2])."""
    th = np.array(theta0, np.float64, copy=True)
    omega = np.ascontiguousarray(omega, np.float64)
    nrec = (nsteps // record_every + 1) if record_every > 0 else 0
    rt = np.zeros((max(nrec, 1), 2), np.float64)
    th10 = np.empty(g.n, np.float64)
    rc = lib().orc_rk4(g._h, _MODES[mode], float(K), float(h), int(nsteps), int(record_every),
                       _p(th), _p(omega), _p(rt) if nrec else None, _p(th10))
    if rc:
        raise ValueError("orc_rk4 failed")
    return th, th10, rt[:nrec]


METHODS = {"euler": 1, "heun": 2, "implicit_midpoint": 3}


def step_method(g: Graph, method, theta0, omega, K, h, nsteps, record_every=1, mode="matvec", fp_tol=1e-13,
                fp_max_iter=50):
    """Euler / Heun / implicit midpoint (NEXT-4); returns (theta_final, r_trace[nrec, 2])."""
    th = np.array(theta0, np.float64, copy=True)
    omega = np.ascontiguousarray(omega, np.float64)
    nrec = (nsteps // record_every + 1) if record_every > 0 else 0
    rt = np.zeros((max(nrec, 1), 2), np.float64)
    rc = lib().orc_step_method(g._h, METHODS[method], _MODES[mode], float(K), float(h), int(nsteps),
                               int(record_every), _p(th), _p(omega), _p(rt) if nrec else None, float(fp_tol),
                               int(fp_max_iter))
    if rc:
        raise ValueError("orc_step_method failed")
    return th, rt[:nrec]


ADAPTIVE_DEFAULTS = dict(h_min=1e-8, h_max=1.0, atol=1e-9, rtol=1e-9, safety=0.9, fac_min=0.2, fac_max=4.0,
                         max_trials=100000)


def integrate_adaptive(g: Graph, theta0, omega, K, t_end, h0, mode="matvec", cap=100000, **ctrl):
    """Variable-step RK4 with step doubling (reading R25).

    Returns (theta(t_end), t[acc], h[acc], rpsi[acc, 2], n_rejected)."""
    c = dict(ADAPTIVE_DEFAULTS, **ctrl)
    th = np.array(theta0, np.float64, copy=True)
    omega = np.ascontiguousarray(omega, np.float64)
    t_out = np.zeros(cap)
    h_out = np.zeros(cap)
    rp = np.zeros((cap, 2))
    rej = ctypes.c_int64(0)
    acc = lib().orc_integrate_adaptive(g._h, _MODES[mode], float(K), float(t_end), float(h0), float(c["h_min"]),
                                       float(c["h_max"]), float(c["atol"]), float(c["rtol"]), float(c["safety"]),
                                       float(c["fac_min"]), float(c["fac_max"]), int(c["max_trials"]), _p(th),
                                       _p(omega), int(cap), _p(t_out), _p(h_out), _p(rp), ctypes.byref(rej))
    if acc < 0:
        raise ValueError(f"orc_integrate_adaptive failed ({acc})")
    k = min(acc, cap)
    return th, t_out[:k], h_out[:k], rp[:k], int(rej.value)


def potential(g: Graph, theta, omega, K):
    """V(theta) of P:474-487 from its definition (uses the graph's scaling)."""
    theta = np.ascontiguousarray(theta, np.float64)
    omega = np.ascontiguousarray(omega, np.float64)
    return float(lib().orc_potential(g._h, float(K), _p(theta), _p(omega)))


def order_parameter(theta):
    theta = np.ascontiguousarray(theta, np.float64)
    out = np.empty(2, np.float64)
    lib().orc_order_parameter(theta.shape[0], _p(theta), _p(out))
    return float(out[0]), float(out[1])
