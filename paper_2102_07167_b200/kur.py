"""Thin Python binding of libkur.so (include/kur.h) — argument marshalling only.

Every step of the hot path runs in libkur's sm_100a kernels; PyTorch only
provides device memory, the current CUDA stream and (for world > 1) the
process group used to broadcast the NCCL id.  There is no CPU fallback: if
libkur.so is missing this module raises ImportError.

Names follow the C ABI: graph_build, rhs, step, order_parameter, permute.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("KUR_LIB") or os.path.join(_HERE, "libkur.so")  # KUR_LIB: tooling builds only
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build() "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

KUR_ONES, KUR_ZEROS = 0, 1
USER_TO_INTERNAL, INTERNAL_TO_USER = 0, 1
STATUS = {0: "KUR_OK", 1: "KUR_ERR_INVALID_ARG", 2: "KUR_ERR_INDEX_RANGE", 3: "KUR_ERR_DUPLICATE_INDEX",
          4: "KUR_ERR_PARTITION", 5: "KUR_ERR_SIZE_MISMATCH", 6: "KUR_ERR_OOM", 7: "KUR_ERR_CUDA",
          8: "KUR_ERR_NCCL", 9: "KUR_ERR_NONFINITE", 10: "KUR_ERR_UNSUPPORTED", 11: "KUR_ERR_STEPSIZE"}

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_d = ctypes.c_double


class GraphDesc(ctypes.Structure):
    _fields_ = [("n", _i64), ("n_comm", _i32), ("community", _p), ("seg_ptr", _p), ("seg_comm", _p),
                ("seg_kind", _p), ("idx_ptr", _p), ("idx", _p), ("dense_threshold", _d),
                ("hot_min", _i32), ("flags", _i32), ("scaling", _i32), ("reserved", _i32)]


class DistDesc(ctypes.Structure):
    _fields_ = [("rank", _i32), ("world", _i32), ("device", _i32), ("nccl_id", _p), ("flags", _i32),
                ("reserved", _i32)]


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("n_comm", _i64), ("rank", _i32), ("world", _i32), ("device", _i32),
                ("rows_per_tile", _i32), ("row_begin", _i64), ("row_end", _i64), ("nnz", _i64),
                ("n_idx", _i64), ("n_idx_hot", _i64), ("n_idx_remote", _i64), ("n_slots_hot", _i64),
                ("n_slots_remote", _i64), ("n_dense_blocks", _i64), ("n_sparse_blocks", _i64),
                ("n_tiles", _i64), ("n_hot_parts", _i64), ("n_window_loads", _i64), ("sincos_per_rhs", _i64),
                ("bytes_per_rhs", _i64), ("bytes_pool", _i64), ("build_seconds", _d), ("remote_pass", _i32),
                ("peer_exchange", _i32)]


class AdaptiveCtrl(ctypes.Structure):
    _fields_ = [("t_end", _d), ("h0", _d), ("h_min", _d), ("h_max", _d), ("atol", _d), ("rtol", _d),
                ("safety", _d), ("fac_min", _d), ("fac_max", _d), ("max_trials", _i64)]


_lib.kur_graph_build.argtypes = [ctypes.POINTER(GraphDesc), ctypes.POINTER(DistDesc), _p, ctypes.POINTER(_p)]
_lib.kur_graph_destroy.argtypes = [_p]
_lib.kur_graph_info.argtypes = [_p, ctypes.POINTER(GraphInfo)]
_lib.kur_graph_permutation.argtypes = [_p, _p]
_lib.kur_permute.argtypes = [_p, _p, _p, _i32, _p]
_lib.kur_rhs.argtypes = [_p, _p, _p, _d, _p, _p]
_lib.kur_step.argtypes = [_p, _p, _p, _d, _d, _i64, _i32, _p, _p]
_lib.kur_order_parameter.argtypes = [_p, _p, _p, _p, _p]
_lib.kur_check.argtypes = [_p, _p]
_lib.kur_potential.argtypes = [_p, _p, _p, _d, _p, _p]
_lib.kur_timing.argtypes = [_p, _i32]
_lib.kur_timing_read.argtypes = [_p, _p]
_lib.kur_nccl_unique_id.argtypes = [_p]
_lib.kur_group_rhs.argtypes = [_p, _i32, _p, _p, _d, _p, _p]
_lib.kur_group_step.argtypes = [_p, _i32, _p, _p, _d, _d, _i64, _i32, _p, _p]
_lib.kur_integrate_adaptive.argtypes = [_p, _p, _p, _d, ctypes.POINTER(AdaptiveCtrl), _i64, _p, _p, _p,
                                        ctypes.POINTER(_i64), ctypes.POINTER(_i64), _p]
_lib.kur_group_integrate_adaptive.argtypes = [_p, _i32, _p, _p, _d, ctypes.POINTER(AdaptiveCtrl), _i64, _p, _p, _p,
                                              ctypes.POINTER(_i64), ctypes.POINTER(_i64), _p]
_lib.kur_step_method.argtypes = [_p, _i32, _p, _p, _d, _d, _i64, _i32, _p, _d, _i32, _p]
_lib.kur_group_step_method.argtypes = [_p, _i32, _i32, _p, _p, _d, _d, _i64, _i32, _p, _d, _i32, _p]
_lib.kur_status_string.restype = ctypes.c_char_p
_lib.kur_status_string.argtypes = [ctypes.c_int]
_lib.kur_last_error.restype = ctypes.c_char_p
for _f in ("kur_graph_build", "kur_graph_destroy", "kur_graph_info", "kur_graph_permutation", "kur_permute",
           "kur_rhs", "kur_step", "kur_order_parameter", "kur_check", "kur_nccl_unique_id", "kur_timing",
           "kur_timing_read", "kur_group_rhs", "kur_group_step", "kur_potential", "kur_step_method",
           "kur_group_step_method", "kur_integrate_adaptive", "kur_group_integrate_adaptive"):
    getattr(_lib, _f).restype = ctypes.c_int

EXPORTED = ("kur_graph_build", "kur_graph_destroy", "kur_graph_info", "kur_graph_permutation", "kur_permute",
            "kur_rhs", "kur_step", "kur_order_parameter", "kur_check", "kur_nccl_unique_id",
            "kur_status_string", "kur_last_error", "kur_timing", "kur_timing_read", "kur_group_rhs",
            "kur_group_step", "kur_potential", "kur_step_method", "kur_group_step_method", "kur_integrate_adaptive",
            "kur_group_integrate_adaptive")
METHODS = {"rk4": 0, "euler": 1, "heun": 2, "implicit_midpoint": 3}


class KurError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _check(st):
    if st != 0:
        raise KurError(st, _lib.kur_last_error().decode(errors="replace"))


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev_vec(x, n, device, name):
    if n == 0 and isinstance(x, torch.Tensor) and x.numel() == 0:
        return ctypes.c_void_p(None)  # a rank without rows
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor")
    if x.dtype != torch.float64 or not x.is_cuda or not x.is_contiguous() or x.numel() != n:
        raise ValueError(f"{name} must be a contiguous CUDA float64 tensor with {n} entries")
    if x.device.index != device:
        raise ValueError(f"{name} is on cuda:{x.device.index}, graph on cuda:{device}")
    return ctypes.c_void_p(x.data_ptr())


def _dev_or_host_vec(x, n, device, name):
    """A device vector as _dev_vec, or a contiguous CPU float64 tensor (host buffer: kur_step
    copies it in and back itself; pinned memory gets the result stored by the final stage)."""
    if isinstance(x, torch.Tensor) and not x.is_cuda:
        if x.dtype != torch.float64 or not x.is_contiguous() or x.numel() != n:
            raise ValueError(f"{name} must be a contiguous float64 tensor with {n} entries")
        return ctypes.c_void_p(x.data_ptr())
    return _dev_vec(x, n, device, name)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_lib.kur_nccl_unique_id(buf))
    return buf.raw


class Graph:
    """kur_graph handle.  Build with ``graph_build``."""

    def __init__(self, handle, device):
        self._h = ctypes.c_void_p(handle)
        self.device = device
        info = GraphInfo()
        _check(_lib.kur_graph_info(self._h, ctypes.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in GraphInfo._fields_}
        self.n = int(info.n)
        self.n_comm = int(info.n_comm)
        self.row_begin = int(info.row_begin)
        self.row_end = int(info.row_end)
        self.n_local = self.row_end - self.row_begin
        perm = np.empty(self.n, np.int32)
        _check(_lib.kur_graph_permutation(self._h, _np_ptr(perm)))
        self.perm = perm  # internal position -> user id

    def refresh_info(self):
        """Re-read kur_graph_info (e.g. peer_exchange after the first group call linked the ranks)."""
        info = GraphInfo()
        _check(_lib.kur_graph_info(self._h, ctypes.byref(info)))
        self.info = {k: getattr(info, k) for k, _ in GraphInfo._fields_}
        return self.info

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.kur_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ----------------------------------------------------------- permutations
    def permute(self, x, direction, out=None, stream=None):
        out = torch.empty_like(x) if out is None else out
        _check(_lib.kur_permute(self._h, _dev_vec(x, self.n, self.device, "in"),
                                _dev_vec(out, self.n, self.device, "out"), direction, _stream(stream)))
        return out

    def to_internal(self, x_user, stream=None):
        """Full-length user-order vector -> full-length internal order (device)."""
        return self.permute(x_user, USER_TO_INTERNAL, stream=stream)

    def to_user(self, x_internal, stream=None):
        return self.permute(x_internal, INTERNAL_TO_USER, stream=stream)

    def local(self, x_internal_full):
        """This rank's rows of a full-length internal-order vector."""
        return x_internal_full[self.row_begin:self.row_end]


FLAG_REMOTE_PASS, FLAG_REMOTE_INLINE = 1 << 16, 2 << 16


def _flags(tile_rows, remote_pass):
    return int(tile_rows) | (0 if remote_pass is None else (FLAG_REMOTE_PASS if remote_pass else FLAG_REMOTE_INLINE))


def graph_build(inst=None, *, dense_threshold=-1.0, hot_min=0, tile_rows=0, remote_pass=None, scaling=None,
                device=None, dist=None, **arrays):
    """kur_graph_build from a kurgen.Instance (or the same arrays as keywords).

    scaling: 0 = uniform K/N (default, or inst.scaling), 1 = degree K/deg_m.
    remote_pass: None = automatic, True/False = force the separate remote-gather pass / inline."""
    src = arrays if inst is None else dict(
        n=inst.n, n_comm=inst.n_comm, community=inst.community, seg_ptr=inst.seg_ptr,
        seg_comm=inst.seg_comm, seg_kind=inst.seg_kind, idx_ptr=inst.idx_ptr, idx=inst.idx)
    if scaling is None:
        scaling = int(getattr(inst, "scaling", 0)) if inst is not None else int(arrays.get("scaling", 0))
    keep = dict(
        community=np.ascontiguousarray(src["community"], np.int32),
        seg_ptr=np.ascontiguousarray(src["seg_ptr"], np.int64),
        seg_comm=np.ascontiguousarray(src["seg_comm"], np.int32),
        seg_kind=np.ascontiguousarray(src["seg_kind"], np.uint8),
        idx_ptr=np.ascontiguousarray(src["idx_ptr"], np.int64),
        idx=np.ascontiguousarray(src["idx"], np.int32))
    desc = GraphDesc(n=int(src["n"]), n_comm=int(src["n_comm"]),
                     community=_np_ptr(keep["community"]), seg_ptr=_np_ptr(keep["seg_ptr"]),
                     seg_comm=_np_ptr(keep["seg_comm"]), seg_kind=_np_ptr(keep["seg_kind"]),
                     idx_ptr=_np_ptr(keep["idx_ptr"]), idx=_np_ptr(keep["idx"]),
                     dense_threshold=float(dense_threshold), hot_min=int(hot_min),
                     flags=_flags(tile_rows, remote_pass), scaling=int(scaling), reserved=0)
    if device is None:
        device = torch.cuda.current_device()
    dd = None
    if dist is not None:
        rank, world, nccl_id = dist[:3]
        flags = int(dist[3]) if len(dist) > 3 else 0
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        dd = DistDesc(rank=rank, world=world, device=device,
                      nccl_id=ctypes.cast(idbuf, _p) if idbuf is not None else None, flags=flags, reserved=0)
    h = ctypes.c_void_p()
    with torch.cuda.device(device):
        _check(_lib.kur_graph_build(ctypes.byref(desc), ctypes.byref(dd) if dd is not None else None,
                                    None, ctypes.byref(h)))
    return Graph(h.value, device)


def rhs(g: Graph, theta, omega, K, out=None, stream=None):
    """dtheta = G(theta) on this rank's rows (internal order, device)."""
    if out is None:
        out = torch.empty_like(theta)
    _check(_lib.kur_rhs(g._h, _dev_vec(theta, g.n_local, g.device, "theta"),
                        _dev_vec(omega, g.n_local, g.device, "omega"), float(K),
                        _dev_vec(out, g.n_local, g.device, "dtheta"), _stream(stream)))
    return out


def step(g: Graph, theta, omega, K, h, nsteps, record_every=0, r_trace=None, stream=None, check=False):
    """nsteps RK4 steps in place on theta (this rank's rows, internal order).

    Host (CPU) tensors are accepted and handed to kur_step as host pointers: the
    library copies theta in and stores the result back (pinned memory: written by the
    last stage through its device mapping) -- the end-to-end path.  The host result is
    complete once the stream is synchronised.  Returns r_trace ([nrec, 2] device
    tensor) or None.
    """
    if record_every and r_trace is None:
        r_trace = torch.zeros((int(nsteps) // int(record_every) + 1, 2), dtype=torch.float64,
                              device=f"cuda:{g.device}")
    rt = ctypes.c_void_p(r_trace.data_ptr()) if r_trace is not None else None
    _check(_lib.kur_step(g._h, _dev_or_host_vec(theta, g.n_local, g.device, "theta"),
                         _dev_or_host_vec(omega, g.n_local, g.device, "omega"), float(K), float(h), int(nsteps),
                         int(record_every), rt, _stream(stream)))
    if check:
        _check(_lib.kur_check(g._h, _stream(stream)))
    return r_trace


def step_method(g: Graph, method, theta, omega, K, h, nsteps, record_every=0, r_trace=None, fp_tol=1e-13,
                fp_max_iter=50, stream=None, check=False):
    """kur_step_method: nsteps of 'rk4' | 'euler' | 'heun' | 'implicit_midpoint' in place on theta."""
    if record_every and r_trace is None:
        r_trace = torch.zeros((int(nsteps) // int(record_every) + 1, 2), dtype=torch.float64,
                              device=f"cuda:{g.device}")
    rt = ctypes.c_void_p(r_trace.data_ptr()) if r_trace is not None else None
    _check(_lib.kur_step_method(g._h, METHODS[method], _dev_or_host_vec(theta, g.n_local, g.device, "theta"),
                                _dev_or_host_vec(omega, g.n_local, g.device, "omega"), float(K), float(h), int(nsteps),
                                int(record_every), rt, float(fp_tol), int(fp_max_iter), _stream(stream)))
    if check:
        _check(_lib.kur_check(g._h, _stream(stream)))
    return r_trace


ADAPTIVE_DEFAULTS = dict(h_min=1e-8, h_max=1.0, atol=1e-9, rtol=1e-9, safety=0.9, fac_min=0.2, fac_max=4.0,
                         max_trials=100000)


def integrate_adaptive(g: Graph, theta, omega, K, t_end, h0, cap=100000, stream=None, **ctrl):
    """kur_integrate_adaptive: variable-step RK4 (step doubling) from t = 0 to t_end, theta in place.

    Returns (t[acc], h[acc], rpsi[acc, 2], n_rejected) as numpy arrays (host)."""
    c = dict(ADAPTIVE_DEFAULTS, **ctrl)
    cc = AdaptiveCtrl(t_end=float(t_end), h0=float(h0), h_min=float(c["h_min"]), h_max=float(c["h_max"]),
                      atol=float(c["atol"]), rtol=float(c["rtol"]), safety=float(c["safety"]),
                      fac_min=float(c["fac_min"]), fac_max=float(c["fac_max"]), max_trials=int(c["max_trials"]))
    t_out, h_out, rp = np.zeros(cap), np.zeros(cap), np.zeros((cap, 2))
    acc, rej = _i64(0), _i64(0)
    _check(_lib.kur_integrate_adaptive(g._h, _dev_vec(theta, g.n_local, g.device, "theta"),
                                       _dev_vec(omega, g.n_local, g.device, "omega"), float(K), ctypes.byref(cc),
                                       int(cap), _np_ptr(t_out), _np_ptr(h_out), _np_ptr(rp), ctypes.byref(acc),
                                       ctypes.byref(rej), _stream(stream)))
    k = min(int(acc.value), cap)
    return t_out[:k], h_out[:k], rp[:k], int(rej.value)


def group_integrate_adaptive(graphs, thetas, omegas, K, t_end, h0, cap=100000, stream=None, **ctrl):
    """kur_group_integrate_adaptive on per-rank local-row device tensors (in place)."""
    c = dict(ADAPTIVE_DEFAULTS, **ctrl)
    cc = AdaptiveCtrl(t_end=float(t_end), h0=float(h0), h_min=float(c["h_min"]), h_max=float(c["h_max"]),
                      atol=float(c["atol"]), rtol=float(c["rtol"]), safety=float(c["safety"]),
                      fac_min=float(c["fac_min"]), fac_max=float(c["fac_max"]), max_trials=int(c["max_trials"]))
    t_out, h_out, rp = np.zeros(cap), np.zeros(cap), np.zeros((cap, 2))
    acc, rej = _i64(0), _i64(0)
    hs = _ptr_array([g._h for g in graphs])
    th = _ptr_array([_dev_vec(t, g.n_local, g.device, "theta").value for g, t in zip(graphs, thetas)])
    om = _ptr_array([_dev_vec(o, g.n_local, g.device, "omega").value for g, o in zip(graphs, omegas)])
    _check(_lib.kur_group_integrate_adaptive(hs, len(graphs), th, om, float(K), ctypes.byref(cc), int(cap),
                                             _np_ptr(t_out), _np_ptr(h_out), _np_ptr(rp), ctypes.byref(acc),
                                             ctypes.byref(rej), _stream(stream)))
    k = min(int(acc.value), cap)
    return t_out[:k], h_out[:k], rp[:k], int(rej.value)


def timing(g: Graph, enable: bool):
    """Enable/disable per-launch CUDA-event timing inside kur_step (clears the record)."""
    _check(_lib.kur_timing(g._h, 1 if enable else 0))


def timing_read(g: Graph):
    """dict(prologue_ms, prologue_n, stage_ms, stage_n, remote_ms, remote_n, launches) of the launches
    recorded since enabling (stage = k_stage or a single-launch trajectory kernel, remote = k_remote)."""
    out = np.zeros(9, np.float64)
    _check(_lib.kur_timing_read(g._h, _np_ptr(out)))
    return dict(prologue_ms=float(out[0]), prologue_n=int(out[1]), stage_ms=float(out[2]), stage_n=int(out[3]),
                remote_ms=float(out[4]), remote_n=int(out[5]), launches=int(out[6]), phase_a_ms=float(out[7]),
                phase_a_n=int(out[8]))


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[p.value if isinstance(p, ctypes.c_void_p) else p for p in ptrs])
    return arr


DIST_PEER_EXCHANGE = 1


def group_build(inst, world, device=None, peer_exchange=False, **kw):
    """world rank handles on ONE device for the single-process group calls (kur_group_*)."""
    fl = DIST_PEER_EXCHANGE if peer_exchange else 0
    return [graph_build(inst, device=device, dist=(r, world, None, fl), **kw) for r in range(world)]


def group_rhs(graphs, thetas, omegas, K, outs=None, stream=None):
    """kur_group_rhs: thetas/omegas/outs are per-rank local-row device tensors."""
    outs = [torch.empty_like(t) for t in thetas] if outs is None else outs
    hs = _ptr_array([g._h for g in graphs])
    th = _ptr_array([_dev_vec(t, g.n_local, g.device, "theta").value for g, t in zip(graphs, thetas)])
    om = _ptr_array([_dev_vec(o, g.n_local, g.device, "omega").value for g, o in zip(graphs, omegas)])
    ou = _ptr_array([_dev_vec(o, g.n_local, g.device, "dtheta").value for g, o in zip(graphs, outs)])
    _check(_lib.kur_group_rhs(hs, len(graphs), th, om, float(K), ou, _stream(stream)))
    return outs


def group_step(graphs, thetas, omegas, K, h, nsteps, record_every=0, stream=None):
    """kur_group_step: in-place RK4 on per-rank local-row device tensors; returns per-rank r_traces."""
    dev = f"cuda:{graphs[0].device}"
    rts = [torch.zeros((int(nsteps) // int(record_every) + 1, 2), dtype=torch.float64, device=dev)
           if record_every else None for _ in graphs]
    hs = _ptr_array([g._h for g in graphs])
    th = _ptr_array([_dev_vec(t, g.n_local, g.device, "theta").value for g, t in zip(graphs, thetas)])
    om = _ptr_array([_dev_vec(o, g.n_local, g.device, "omega").value for g, o in zip(graphs, omegas)])
    rt = _ptr_array([r.data_ptr() if r is not None else None for r in rts]) if record_every else None
    _check(_lib.kur_group_step(hs, len(graphs), th, om, float(K), float(h), int(nsteps), int(record_every), rt,
                               _stream(stream)))
    return rts


def group_step_method(graphs, method, thetas, omegas, K, h, nsteps, record_every=0, fp_tol=1e-13, fp_max_iter=50,
                      stream=None):
    """kur_group_step_method on per-rank local-row device tensors; returns per-rank r_traces."""
    dev = f"cuda:{graphs[0].device}"
    rts = [torch.zeros((int(nsteps) // int(record_every) + 1, 2), dtype=torch.float64, device=dev)
           if record_every else None for _ in graphs]
    hs = _ptr_array([g._h for g in graphs])
    th = _ptr_array([_dev_vec(t, g.n_local, g.device, "theta").value for g, t in zip(graphs, thetas)])
    om = _ptr_array([_dev_vec(o, g.n_local, g.device, "omega").value for g, o in zip(graphs, omegas)])
    rt = _ptr_array([r.data_ptr() if r is not None else None for r in rts]) if record_every else None
    _check(_lib.kur_group_step_method(hs, len(graphs), METHODS[method], th, om, float(K), float(h), int(nsteps),
                                      int(record_every), rt, float(fp_tol), int(fp_max_iter), _stream(stream)))
    return rts


def potential(g: Graph, theta, omega, K, stream=None):
    """V(theta) as a device tensor [1]."""
    out = torch.empty(1, dtype=torch.float64, device=f"cuda:{g.device}")
    _check(_lib.kur_potential(g._h, _dev_vec(theta, g.n_local, g.device, "theta"),
                              _dev_vec(omega, g.n_local, g.device, "omega"), float(K),
                              ctypes.c_void_p(out.data_ptr()), _stream(stream)))
    return out


def check(g: Graph, stream=None):
    _check(_lib.kur_check(g._h, _stream(stream)))


def order_parameter(g: Graph, theta, local=False, stream=None):
    """(r, psi) device tensor [2]; with local=True also [n_comm, 2] local (r_b, psi_b)."""
    out = torch.empty(2, dtype=torch.float64, device=f"cuda:{g.device}")
    loc = torch.empty((g.n_comm, 2), dtype=torch.float64, device=f"cuda:{g.device}") if local else None
    _check(_lib.kur_order_parameter(g._h, _dev_vec(theta, g.n_local, g.device, "theta"),
                                    ctypes.c_void_p(out.data_ptr()),
                                    ctypes.c_void_p(loc.data_ptr()) if loc is not None else None,
                                    _stream(stream)))
    return (out, loc) if local else out


# ------------------------------------------------------------------ host-only plan introspection
_lib.kur_plan_build.argtypes = [ctypes.POINTER(GraphDesc), _i32, _i32, _i32, ctypes.POINTER(_p)]
_lib.kur_plan_sizes.argtypes = [_p, _p]
_lib.kur_plan_export.argtypes = [_p] + [_p] * 7
_lib.kur_plan_destroy.argtypes = [_p]
_lib.kur_plan_tiles.argtypes = [_p, _p, _p]
for _f in ("kur_plan_build", "kur_plan_sizes", "kur_plan_export", "kur_plan_destroy", "kur_plan_tiles"):
    getattr(_lib, _f).restype = ctypes.c_int
EXPORTED = EXPORTED + ("kur_plan_build", "kur_plan_sizes", "kur_plan_export", "kur_plan_destroy", "kur_plan_tiles")


def _desc_from(inst, dense_threshold=-1.0, hot_min=0, tile_rows=0):
    keep = dict(
        community=np.ascontiguousarray(inst.community, np.int32),
        seg_ptr=np.ascontiguousarray(inst.seg_ptr, np.int64),
        seg_comm=np.ascontiguousarray(inst.seg_comm, np.int32),
        seg_kind=np.ascontiguousarray(inst.seg_kind, np.uint8),
        idx_ptr=np.ascontiguousarray(inst.idx_ptr, np.int64),
        idx=np.ascontiguousarray(inst.idx, np.int32))
    desc = GraphDesc(n=int(inst.n), n_comm=int(inst.n_comm), community=_np_ptr(keep["community"]),
                     seg_ptr=_np_ptr(keep["seg_ptr"]), seg_comm=_np_ptr(keep["seg_comm"]),
                     seg_kind=_np_ptr(keep["seg_kind"]), idx_ptr=_np_ptr(keep["idx_ptr"]),
                     idx=_np_ptr(keep["idx"]), dense_threshold=float(dense_threshold),
                     hot_min=int(hot_min), flags=int(tile_rows), scaling=int(getattr(inst, "scaling", 0)),
                     reserved=0)
    return desc, keep


def plan_export(inst, *, rank=0, world=1, sm_count=148, dense_threshold=-1.0, hot_min=0, tile_rows=0):
    """Host-only: build the block plan and decode its stored layout (see kur.h)."""
    desc, keep = _desc_from(inst, dense_threshold, hot_min, tile_rows)
    h = ctypes.c_void_p()
    _check(_lib.kur_plan_build(ctypes.byref(desc), rank, world, sm_count, ctypes.byref(h)))
    try:
        sz = np.zeros(16, np.int64)
        _check(_lib.kur_plan_sizes(h, _np_ptr(sz)))
        n, C, nl, rb, ne, nd, nt, rpt_rows, nnz, w = (int(x) for x in sz[:10])
        out = dict(n=n, n_comm=C, n_local=nl, row_begin=rb, n_tiles=nt, rows_per_tile=rpt_rows, nnz=nnz,
                   perm=np.empty(n, np.int32), D_ptr=np.empty(C + 1, np.int32),
                   D_idx=np.empty(max(nd, 1), np.int32), row_ptr=np.empty(nl + 1, np.int64),
                   cols=np.empty(max(ne, 1), np.int32), neg=np.empty(max(ne, 1), np.int8),
                   shard_row0=np.empty(w + 1, np.int32))
        _check(_lib.kur_plan_export(h, *[ctypes.c_void_p(out[k].ctypes.data) for k in
                                         ("perm", "D_ptr", "D_idx", "row_ptr", "cols", "neg", "shard_row0")]))
        out["D_idx"] = out["D_idx"][:nd]
        out["cols"] = out["cols"][:ne]
        out["neg"] = out["neg"][:ne]
        _check(_lib.kur_plan_sizes(h, _np_ptr(sz)))
        out.update(conflicts=int(sz[10]), slots_hot=int(sz[11]), idx_hot=int(sz[12]), slots_remote=int(sz[13]),
                   idx_remote=int(sz[14]), window_loads=int(sz[15]))
        tiles = np.zeros((max(nt, 1), 7), np.int32)
        _check(_lib.kur_plan_tiles(h, ctypes.c_void_p(tiles.ctypes.data), None))
        pw = np.zeros(max(int(tiles[:nt, 3].sum()), 1), np.int32)
        _check(_lib.kur_plan_tiles(h, ctypes.c_void_p(tiles.ctypes.data), ctypes.c_void_p(pw.ctypes.data)))
        out["tiles"] = tiles[:nt]
        out["part_window"] = pw[:int(tiles[:nt, 3].sum())]
        return out
    finally:
        _lib.kur_plan_destroy(h)
