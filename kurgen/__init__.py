"""kurgen — seeded synthetic instances for the Kuramoto-on-graphs hot path.

This module is the ONE piece shared by the oracle tests, the GPU parity tests
and bench.py: it draws counter-based random numbers (SplitMix64, reading R18
in DESIGN.md) and emits adjacency patterns in the row-segmented layout of
``include/kur.h`` (``kur_graph_desc``).  It contains none of the method's
arithmetic — no trigonometry of phases, no sums over neighbours, no block
sums — so sharing it does not couple the oracle to the CUDA path.

Workload recipes follow BASELINE.json ``configs`` (the paper's own workloads
are synthetic too: uniform phases, random frequencies, random threshold/block
matrices).
"""
from __future__ import annotations

import ctypes
import hashlib
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_LIB = os.path.join(_HERE, "libkurgen.so")

KUR_ONES = 0
KUR_ZEROS = 1

# named counter streams (reading R18)
S_OMEGA, S_THETA0, S_SIZES, S_PDRAW, S_PAIRS, S_PERM = 1, 2, 3, 4, 5, 6
S_EDGES = 1 << 40
SEED_BASE = 2102071670  # seed_cfg = SEED_BASE + cfg


def _load():
    if not os.path.exists(_LIB):
        subprocess.run(["make", "-s", "-C", _ROOT, "kurgen/libkurgen.so"], check=True)
    lib = ctypes.CDLL(_LIB)
    d, i64, u64 = ctypes.c_double, ctypes.c_int64, ctypes.c_uint64
    p = ctypes.c_void_p
    lib.kg_uniform.argtypes = [u64, u64, i64, d, d, p]
    lib.kg_normal.argtypes = [u64, u64, i64, d, d, p]
    lib.kg_cauchy_trunc.argtypes = [u64, u64, i64, d, p]
    lib.kg_permutation.argtypes = [u64, u64, i64, p]
    lib.kg_bits.argtypes = [u64, u64, i64, p]
    lib.kg_sbm_count.argtypes = [i64, ctypes.c_int32, p, p, p, u64, u64, p]
    lib.kg_sbm_count.restype = i64
    lib.kg_sbm_fill.argtypes = [i64, ctypes.c_int32, p, p, p, p, u64, u64, p, p, p]
    lib.kg_sbm_segments.argtypes = [i64, ctypes.c_int32, p, p, p, p, p, p, p, p, p]
    lib.kg_sbm_segments.restype = i64
    return lib


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = _load()
    return _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


# ------------------------------------------------------------------ scalars
def uniform(seed, stream, n, lo=0.0, hi=1.0):
    out = np.empty(n, np.float64)
    lib().kg_uniform(seed, stream, n, lo, hi, _ptr(out))
    return out


def normal(seed, stream, n, mu=0.0, sigma=1.0):
    out = np.empty(n, np.float64)
    lib().kg_normal(seed, stream, n, mu, sigma, _ptr(out))
    return out


def cauchy_trunc(seed, stream, n, limit):
    out = np.empty(n, np.float64)
    lib().kg_cauchy_trunc(seed, stream, n, limit, _ptr(out))
    return out


def permutation(seed, stream, n):
    out = np.empty(n, np.int32)
    lib().kg_permutation(seed, stream, n, _ptr(out))
    return out


def raw_bits(seed, stream, n):
    out = np.empty(n, np.uint64)
    lib().kg_bits(seed, stream, n, _ptr(out))
    return out


# ------------------------------------------------------------------ instance
@dataclass
class Instance:
    """A graph in user numbering plus the ODE data (kur_graph_desc + omega, theta0)."""

    name: str
    n: int
    n_comm: int
    community: np.ndarray  # int32[n]  community label of user node u
    seg_ptr: np.ndarray  # int64[n+1]
    seg_comm: np.ndarray  # int32[nseg]
    seg_kind: np.ndarray  # uint8[nseg]  KUR_ONES / KUR_ZEROS
    idx_ptr: np.ndarray  # int64[nseg+1]
    idx: np.ndarray  # int32[nidx]  user column ids
    omega: np.ndarray  # float64[n]
    theta0: np.ndarray  # float64[n]
    K: float = 1.0
    h: float = 0.01
    nsteps: int = 10
    record_every: int = 1
    seed: int = 0
    scaling: int = 0  # 0: uniform M_m = N; 1: degree M_m = sum_l A_ml
    meta: dict = field(default_factory=dict)

    @property
    def nseg(self):
        return int(self.seg_comm.shape[0])

    @property
    def nidx(self):
        return int(self.idx.shape[0])

    def sha256(self):
        h = hashlib.sha256()
        for a in (self.community, self.seg_ptr, self.seg_comm, self.seg_kind,
                  self.idx_ptr, self.idx, self.omega, self.theta0):
            h.update(np.ascontiguousarray(a).view(np.uint8).data)
        h.update(repr((self.n, self.n_comm, self.K, self.h, self.nsteps,
                       self.record_every)).encode())
        return h.hexdigest()

    def dense(self):
        """Expand to a dense 0/1 matrix (tests only; diagonal left 0)."""
        n = self.n
        A = np.zeros((n, n), np.uint8)
        members = [np.flatnonzero(self.community == c) for c in range(self.n_comm)]
        for u in range(n):
            for s in range(self.seg_ptr[u], self.seg_ptr[u + 1]):
                lst = self.idx[self.idx_ptr[s]:self.idx_ptr[s + 1]]
                b = self.seg_comm[s]
                if self.seg_kind[s] == KUR_ONES:
                    A[u, lst] = 1
                else:
                    A[u, members[b]] = 1
                    A[u, lst] = 0
            A[u, u] = 0
        return A


def sbm(sizes, P, seed, *, omega=("normal", 0.0, 1.0), K=1.0, h=0.01, nsteps=10,
        record_every=1, name="sbm", permute=True):
    """Symmetric stochastic block model with planted partition (reading R14).

    sizes: community sizes (internal contiguous order); P: symmetric C x C
    probabilities.  Labels are randomly permuted when ``permute`` (R16).
    """
    sizes = np.asarray(sizes, np.int64)
    C = int(sizes.shape[0])
    P = np.ascontiguousarray(np.asarray(P, np.float64).reshape(C, C))
    assert np.allclose(P, P.T), "P must be symmetric"
    n = int(sizes.sum())
    coff = np.zeros(C + 1, np.int64)
    coff[1:] = np.cumsum(sizes)
    perm = permutation(seed, S_PERM, n) if permute else np.arange(n, dtype=np.int32)
    labels = np.empty(n, np.int32)
    labels[perm] = np.repeat(np.arange(C, dtype=np.int32), sizes)
    L = lib()
    row_cnt = np.zeros(n, np.int64)
    tot = L.kg_sbm_count(n, C, _ptr(coff), _ptr(P), _ptr(perm), seed, S_EDGES, _ptr(row_cnt))
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(row_cnt, out=row_ptr[1:])
    assert row_ptr[-1] == tot
    assert tot < 2**31 * 4, "instance too large"
    cols = np.empty(tot, np.int32)
    scratch = np.empty(n, np.int64)
    L.kg_sbm_fill(n, C, _ptr(coff), _ptr(P), _ptr(perm), _ptr(labels), seed, S_EDGES,
                  _ptr(row_ptr), _ptr(cols), _ptr(scratch))
    seg_cnt = np.zeros(n, np.int64)
    nseg = L.kg_sbm_segments(n, C, _ptr(labels), _ptr(P), _ptr(row_ptr), _ptr(cols),
                             _ptr(seg_cnt), None, None, None, None)
    seg_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(seg_cnt, out=seg_ptr[1:])
    seg_comm = np.empty(nseg, np.int32)
    seg_kind = np.empty(nseg, np.uint8)
    idx_ptr = np.empty(nseg + 1, np.int64)
    L.kg_sbm_segments(n, C, _ptr(labels), _ptr(P), _ptr(row_ptr), _ptr(cols),
                      _ptr(seg_cnt), _ptr(seg_ptr), _ptr(seg_comm), _ptr(seg_kind),
                      _ptr(idx_ptr))
    idx_ptr[nseg] = tot
    del scratch, row_cnt
    kind, a, b = omega
    if kind == "normal":
        om = normal(seed, S_OMEGA, n, a, b)
    elif kind == "cauchy":
        om = cauchy_trunc(seed, S_OMEGA, n, a)
    elif kind == "zero":
        om = np.zeros(n)
    else:
        raise ValueError(kind)
    th = uniform(seed, S_THETA0, n, 0.0, 2.0 * math.pi)
    return Instance(name=name, n=n, n_comm=C, community=labels, seg_ptr=seg_ptr,
                    seg_comm=seg_comm, seg_kind=seg_kind, idx_ptr=idx_ptr, idx=cols,
                    omega=om, theta0=th, K=K, h=h, nsteps=nsteps,
                    record_every=record_every, seed=seed,
                    meta={"sizes": sizes.tolist() if C <= 4096 else None,
                          "perm_internal_to_user": perm})


def complete_graph(n, seed, *, omega=("normal", 0.0, 1.0), K=1.0, h=0.01, nsteps=10,
                   record_every=1, name="complete"):
    """A = all-ones minus identity: one community, one empty KUR_ZEROS segment per row."""
    return sbm([n], [[1.0]], seed, omega=omega, K=K, h=h, nsteps=nsteps,
               record_every=record_every, name=name, permute=False)


def _config4_blocks(seed, N=262144, C=64):
    """Config 4 sizes and probabilities (readings R13, R15)."""
    u = uniform(seed, S_SIZES, C)
    x = np.exp(np.log(512.0) + u * (np.log(16384.0) - np.log(512.0)))
    q = N * x / x.sum()
    sizes = np.floor(q).astype(np.int64)
    rem = N - int(sizes.sum())
    order = np.argsort(-(q - sizes), kind="stable")
    sizes[order[:rem]] += 1
    assert sizes.sum() == N
    pick = raw_bits(seed, S_PDRAW, C) % np.uint64(3)
    pin = np.array([0.99, 0.6, 0.05])[pick.astype(np.int64)]
    P = np.full((C, C), 1e-4)
    np.fill_diagonal(P, pin)
    bits = raw_bits(seed, S_PAIRS, 4096)
    chosen, k = [], 0
    while len(chosen) < 8:
        a = int(bits[k] % np.uint64(C)); b = int(bits[k + 1] % np.uint64(C)); k += 2
        if a == b:
            continue
        pr = (min(a, b), max(a, b))
        if pr not in chosen:
            chosen.append(pr)
    for a, b in chosen:
        P[a, b] = P[b, a] = 0.9
    return sizes, P, chosen


def config(k):
    """BASELINE.json configs[k-1] (k = 1..5) as a seeded synthetic instance."""
    seed = SEED_BASE + k
    if k == 1:
        return complete_graph(1000, seed, omega=("normal", 0.0, 1.0), K=2.0, h=0.01,
                              nsteps=50, record_every=1, name="cfg1-complete-N1000")
    if k == 2:
        return complete_graph(1 << 20, seed, omega=("cauchy", 10.0, None), K=3.0, h=0.01,
                              nsteps=1000, record_every=10, name="cfg2-complete-N2^20")
    if k == 3:
        C = 16
        P = np.full((C, C), 0.001)
        np.fill_diagonal(P, 0.95)
        return sbm([4096] * C, P, seed, omega=("normal", 0.0, 1.0), K=4.0, h=0.005,
                   nsteps=200, name="cfg3-sbm-16x4096")
    if k == 4:
        sizes, P, pairs = _config4_blocks(seed)
        inst = sbm(sizes, P, seed, omega=("normal", 0.0, 0.5), K=5.0, h=0.005, nsteps=200,
                   name="cfg4-hetero-sbm-64")
        inst.meta["dense_pairs"] = pairs
        return inst
    if k == 5:
        C = 256
        P = np.full((C, C), 2e-6)
        np.fill_diagonal(P, 0.98)
        return sbm([16384] * C, P, seed, omega=("normal", 0.0, 1.0), K=4.0, h=0.01,
                   nsteps=100, name="cfg5-sbm-256x16384")
    raise ValueError(k)


def from_dense(A, labels, *, kind="auto", seed=0, omega=None, theta0=None, K=1.0, h=0.01,
               nsteps=10, record_every=1, name="dense", scaling=0, self_loops=False):
    """Encode a dense 0/1 matrix with community labels.

    kind: 'ones' (plain CSR), 'zeros' (every block as KUR_ZEROS), 'auto'
    (per row/block whichever list is shorter), 'random' (coin per segment).
    The diagonal is ignored unless self_loops: then A[u,u] = 1 is stored by
    listing u in a KUR_ONES segment of its own community (reading R22; it only
    matters for the degree scaling).  Small sizes only (tests).
    """
    A = np.asarray(A).astype(np.uint8)
    n = A.shape[0]
    labels = np.asarray(labels, np.int32)
    C = int(labels.max()) + 1 if n else 0
    members = [np.flatnonzero(labels == c).astype(np.int32) for c in range(C)]
    coin = raw_bits(seed + 99, 7, max(1, n * max(C, 1)))
    seg_ptr = [0]
    seg_comm, seg_kind, idx_ptr, idx = [], [], [0], []
    for u in range(n):
        for b in range(C):
            m = members[b]
            m_off = m[m != u]
            row = A[u, m_off]
            ones = m_off[row == 1]
            zeros = m_off[row == 0]
            loop = bool(self_loops and b == labels[u] and A[u, u])
            if loop:
                kd = KUR_ONES
                ones = np.sort(np.concatenate([ones, [u]])).astype(np.int32)
            elif kind == "ones":
                kd = KUR_ONES
            elif kind == "zeros":
                kd = KUR_ZEROS
            elif kind == "auto":
                kd = KUR_ZEROS if len(zeros) < len(ones) else KUR_ONES
            elif kind == "random":
                kd = int(coin[u * C + b] & np.uint64(1))
            else:
                raise ValueError(kind)
            lst = ones if kd == KUR_ONES else zeros
            if kd == KUR_ONES and len(lst) == 0:
                continue
            seg_comm.append(b)
            seg_kind.append(kd)
            idx.extend(lst.tolist())
            idx_ptr.append(len(idx))
        seg_ptr.append(len(seg_comm))
    om = normal(seed, S_OMEGA, n) if omega is None else np.asarray(omega, np.float64)
    th = uniform(seed, S_THETA0, n, 0.0, 2 * math.pi) if theta0 is None else np.asarray(theta0, np.float64)
    return Instance(name=name, n=n, n_comm=C, community=labels,
                    seg_ptr=np.asarray(seg_ptr, np.int64),
                    seg_comm=np.asarray(seg_comm, np.int32),
                    seg_kind=np.asarray(seg_kind, np.uint8),
                    idx_ptr=np.asarray(idx_ptr, np.int64), idx=np.asarray(idx, np.int32),
                    omega=om.copy(), theta0=th.copy(), K=K, h=h, nsteps=nsteps,
                    record_every=record_every, seed=seed, scaling=scaling)


def random_dense(n, C, seed, p_in=0.8, p_out=0.1, symmetric=True):
    """Small random block-structured 0/1 matrix + labels (tests)."""
    labels = (raw_bits(seed, S_SIZES, n) % np.uint64(max(C, 1))).astype(np.int32) if C > 1 \
        else np.zeros(n, np.int32)
    u = uniform(seed, S_PAIRS, n * n).reshape(n, n)
    same = labels[:, None] == labels[None, :]
    A = (u < np.where(same, p_in, p_out)).astype(np.uint8)
    if symmetric:
        A = np.triu(A, 1)
        A = A + A.T
    np.fill_diagonal(A, 0)
    return A, labels
