#!/usr/bin/env python
"""bench.py — Kuramoto-on-graphs RHS through localised order parameters +
classical RK4 on B200 (BASELINE.json metric: RHS evals/s and achieved HBM
GB/s; RK4 steps/s at 1/2/4/8 GPUs).

A "step" is one classical RK4 step of the whole hot path (SURVEY.md §8(a)
a1-a6: 4 RHS evaluations through the block sums and the complement /
non-zero lists, the fused RK updates, and the recorded order parameter) over
the configured synthetic instance (default: BASELINE configs[4] = config 5,
N = 2^22, the graph the metric's 1/2/4/8-GPU numbers are quoted on; it fits
one GPU).  ``value`` = RHS evaluations per second of the whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl kur|reference]

Prints ONE JSON line on rank 0.  The timed region is bracketed by a barrier
and torch.cuda.synchronize() and timed with CUDA events on the launching
stream; multi-GPU times are the max over ranks.  The inputs (index pool of
several GB) are far larger than the 126 MB L2, so no flush is needed.
"""
import argparse
import json
import math
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Kuramoto RHS evals/s (fused RK4 stages; achieved HBM GB/s and RK4 steps/s reported alongside)"
UNIT = "RHS/s"


def _measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _ncu_traffic(cfg):
    """DRAM bytes of one RHS evaluation (k_remote + k_stage) from the committed ncu captures, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        v = t.get(f"cfg{cfg}")
        return None if v is None else float(v["dram_bytes_per_rhs"])
    except Exception:
        return None


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device_index):
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self.samples, self.reasons = [], 0
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml unavailable"], "samples": 0}
        names = [n for b, n in self.REASONS.items() if self.reasons & b and b != 0x1]
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def _host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "omp_num_threads": os.environ.get("OMP_NUM_THREADS")}


def _relaunch_distributed(n):
    """`bench.py --gpus N` without a torchrun environment: run N ranks (one per GPU) under
    torch.distributed.run on this node and return its exit code."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_rhs_rate(inst, rows_sample, mode="matvec", threads=None, reps=1):
    """Oracle RHS evaluations/s extrapolated from a bounded row sample (rows_sample None: the whole
    graph), median of `reps` timings, on `threads` host threads (None: all).  Test infrastructure:
    bench.py's cpu_baseline leg only."""
    import oracle
    og = oracle.Graph(inst)
    all_threads = oracle.num_threads()
    oracle.set_num_threads(threads or all_threads)
    try:
        rows = None if rows_sample is None else np.ascontiguousarray(rows_sample, np.int64)
        nrow = inst.n if rows is None else rows.size
        oracle.rhs(og, inst.theta0, inst.omega, inst.K, mode=mode, rows=None if rows is None else rows[:64])  # warm
        dts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            oracle.rhs(og, inst.theta0, inst.omega, inst.K, mode=mode, rows=rows)
            dts.append(time.perf_counter() - t0)
        dt = float(np.median(dts))
        return 1.0 / (dt * inst.n / nrow), dt, oracle.num_threads()
    finally:
        oracle.set_num_threads(all_threads)


# SURVEY 8(d) / BASELINE.md §3 oracle protocol per config: (mode, rows sampled at all cores, rows at 1 core).
# None = the whole graph.  cfg2's naive mode costs N per row (1.1e12 sines per RHS): timed per row on 256
# sampled rows and reported "per row", not extrapolated into the headline; its headline is the O(N) op form.
def _cpu_protocol_plan(inst, cfg):
    comm_rows = lambda k: np.flatnonzero(np.isin(inst.community, np.arange(0, inst.n_comm,
                                                                           max(1, inst.n_comm // k))[:k]))
    if cfg == 1:
        return [("naive", None, None), ("op", None, None)]
    if cfg == 2:
        return [("op", None, None), ("naive", np.arange(0, inst.n, inst.n // 256)[:256], "per_row")]
    if cfg == 3:
        return [("matvec", None, None), ("naive", comm_rows(2), None)]
    if cfg == 4:
        return [("matvec", comm_rows(16), None)]
    return [("matvec", comm_rows(128), comm_rows(1))]


def cpu_protocol(inst, cfg):
    """The oracle timed on this host at all cores and at 1 core (bounded samples), per mode."""
    out, head = [], None
    for mode, rows, extra in _cpu_protocol_plan(inst, cfg):
        r_all, dt_all, cores = cpu_oracle_rhs_rate(inst, rows, mode, reps=3 if (rows is None and inst.n <= 70000) else 1)
        rows1 = rows
        if extra is not None and not isinstance(extra, str):
            rows1 = extra
        r_one, dt_one, _ = cpu_oracle_rhs_rate(inst, rows1, mode, threads=1)
        nrow = inst.n if rows is None else rows.size
        rec = {"mode": mode, "rows": nrow, "rhs_per_s_all_cores": r_all, "rhs_per_s_1_core": r_one,
               "steps_per_s_all_cores": r_all / 4.0, "steps_per_s_1_core": r_one / 4.0, "cores": cores,
               "seconds": dt_all + dt_one}
        if isinstance(extra, str) and extra == "per_row":
            rec = {"mode": mode, "rows": nrow, "unit": "rows/s (not extrapolated)",
                   "rows_per_s_all_cores": r_all * inst.n, "rows_per_s_1_core": r_one * inst.n, "cores": cores,
                   "seconds": dt_all + dt_one}
        elif head is None:
            head = (rec, nrow)
        out.append(rec)
    rec, nrow = head
    return {"value": rec["rhs_per_s_all_cores"], "unit": UNIT, "cores": rec["cores"], "kind": "oracle",
            "sample": f"oracle {rec['mode']} RHS on {nrow} of {inst.n} rows" +
                      ("" if nrow == inst.n else f", extrapolated x{inst.n / nrow:.1f}") +
                      "; steps/s = RHS/s / 4 (an RK4 step is 4 RHS evaluations plus O(N) updates)",
            "protocol": out, "host": _host_info()}


def _sample_rows(inst, cfg):
    # whole communities (the oracle's per-row cost is the row's degree, so sample real rows)
    if inst.n_comm > 1:
        k = {3: 16, 4: 16, 5: 128}.get(cfg, 4)  # ~10 s of host work for the default (cfg5) line
        comms = np.arange(0, inst.n_comm, max(1, inst.n_comm // k))[:k]
        return np.flatnonzero(np.isin(inst.community, comms))
    return np.arange(0, inst.n, max(1, inst.n // 20000))


def run_reference(args):
    """--impl reference: the oracle (the only reference this tier has), timed on host cores."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    import kurgen
    inst = kurgen.config(args.config)
    rows = _sample_rows(inst, args.config)
    if args.config == 5:
        rows = rows[: 16384]  # one community per step keeps the whole run within minutes
    rates = []
    for i in range(args.warmup + args.steps):
        r, dt, cores = cpu_oracle_rhs_rate(inst, rows)
        if i >= args.warmup:
            rates.append(r)
    val = float(np.median(rates))
    sample = f"matvec RHS on {rows.size} of {inst.n} rows per step, extrapolated x{inst.n / rows.size:.1f}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 4000.0 / val, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": inst.name, "n": inst.n, "n_comm": inst.n_comm, "nnz_directed": None},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="kur", choices=["kur", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--tile-rows", type=int, default=0, help="tuning: force the tile size (rows)")
    ap.add_argument("--hot-min", type=int, default=0, help="tuning: window staging threshold")
    ap.add_argument("--remote-pass", default="auto", choices=["auto", "on", "off"],
                    help="tuning: force the separate k_remote pass on/off")
    ap.add_argument("--peer-exchange", action="store_true",
                    help="N > 1: fused peer-store exchange from the stage kernel instead of ncclAllGather")
    ap.add_argument("--dense-threshold", type=float, default=-1.0,
                    help="ablation (SURVEY 8(d)): 0 forces direct summation (plain CSR), <0 the paper's rule")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch_distributed(args.gpus))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}: one rank per GPU")
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import kurgen
    from paper_2102_07167_b200 import kur

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        # NCCL's INIT lines (communicator size and rank of every process) on stderr, so the rank
        # count is verifiable while stdout keeps the one JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    t0 = time.perf_counter()
    inst = kurgen.config(args.config)
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    rp = {"auto": None, "on": True, "off": False}[args.remote_pass]
    if world > 1:
        obj = [kur.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        g = kur.graph_build(inst, device=local, dist=(rank, world, obj[0], kur.DIST_PEER_EXCHANGE if
                                                      args.peer_exchange else 0), tile_rows=args.tile_rows,
                            hot_min=args.hot_min, dense_threshold=args.dense_threshold, remote_pass=rp)
    else:
        g = kur.graph_build(inst, device=local, tile_rows=args.tile_rows, hot_min=args.hot_min,
                            dense_threshold=args.dense_threshold, remote_pass=rp)
    build_s = time.perf_counter() - t0
    info = g.info
    th = g.local(g.to_internal(torch.from_numpy(inst.theta0).to(dev))).clone()
    om = g.local(g.to_internal(torch.from_numpy(inst.omega).to(dev))).clone()
    K, h = inst.K, inst.h
    stream = torch.cuda.current_stream()

    # ---- warm-up
    kur.step(g, th, om, K, h, args.warmup, 1, check=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    # ---- timed region: exactly K RK4 steps (one kur_step call), no per-launch instrumentation
    r_trace = torch.zeros((args.steps + 1, 2), dtype=torch.float64, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        kur.step(g, th, om, K, h, args.steps, 1, r_trace=r_trace)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kur.check(g)
    r_final = float(r_trace[-1, 0].item())
    # ---- per-kernel breakdown (roofline): the same K steps again with a CUDA event pair around every
    # launch on the launching stream (kur_timing); not part of `value`
    if world > 1:
        dist.barrier()
    kur.timing(g, True)
    kur.step(g, th, om, K, h, args.steps, 1, r_trace=r_trace)
    torch.cuda.synchronize()
    tm = kur.timing_read(g)
    kur.timing(g, False)
    if world > 1:
        t = torch.tensor([ms, tm["stage_ms"], tm["remote_ms"]], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t[0].item())
        tm["stage_ms"] = float(t[1].item())
        tm["remote_ms"] = float(t[2].item())
    ms_per_step = ms / args.steps
    rhs_per_s = 4.0 * args.steps / (ms / 1e3)
    kstage_ms = tm["stage_ms"] / max(tm["stage_n"], 1)
    kremote_ms = tm["remote_ms"] / max(tm["stage_n"], 1)
    stage_ms = kstage_ms + kremote_ms  # one RHS evaluation = [k_remote +] k_stage
    # world 1 with the remote pass: k_stage overlaps k_remote's tail (programmatic dependent launch), so
    # the library times the pair with ONE event pair (an event between them would serialise it)
    overlapped = bool(info["remote_pass"]) and tm["remote_n"] == 0 and tm["stage_n"] > 0

    # ---- roofline of the dominant kernel (the fused RK stage = one RHS evaluation).
    # Algorithmic bytes per launch = SURVEY.md §8(d)'s per-unit figure: B_rhs = 16 N (z) + 4 n_idx
    # (int32 lists) + 8 N (row offsets) + 8 N (omega), plus 24 N for the fused RK stage (theta_n read,
    # acc read/write), N = this rank's rows.  The bytes THIS layout must move (2-byte
    # window-local slots, no row offsets, z written once) are reported beside it as kernel_bytes.
    peak, peak_src = _measured_peaks()
    n_loc = int(info["row_end"] - info["row_begin"])
    bytes_launch = 56 * n_loc + 4 * int(info["n_idx"])
    kernel_bytes = int(info["bytes_per_rhs"])
    achieved = bytes_launch / (stage_ms / 1e3) / 1e9
    traffic = _ncu_traffic(args.config) if world == 1 else None  # the capture is a 1-GPU launch
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "peak_source": peak_src,
                "kernel": ("k_remote + k_stage" if info["remote_pass"] else "k_stage") + " (one RHS evaluation = "
                          "one fused RK4 stage)",
                "bytes_per_launch": bytes_launch,
                "bytes_formula": "SURVEY 8(d): 16N z + 4 n_idx + 8N offsets + 8N omega + 24N RK stage",
                "avg_launch_ms": stage_ms, "k_stage_ms": None if overlapped else kstage_ms,
                "k_remote_ms": None if overlapped else kremote_ms,
                "remote_overlap": ("k_remote + k_stage timed as one event pair: k_stage is launched as k_remote's "
                                   "programmatic dependent and waits for it only before its finalize; the per-"
                                   "kernel split is in the ncu launch list") if overlapped else None,
                "stage_share_of_step": (tm["stage_ms"] + tm["remote_ms"]) / ms if ms > 0 else None,
                "timing": "avg_launch_ms from a second K-step run with per-launch CUDA events; value and "
                          "ms_per_step from the uninstrumented run",
                "kernel_bytes_per_launch": kernel_bytes,
                "kernel_bytes_gbs": kernel_bytes / (stage_ms / 1e3) / 1e9,
                "kernel_bytes_frac": kernel_bytes / (stage_ms / 1e3) / 1e9 / peak,
                "traffic_gbs": None if traffic is None else traffic / (stage_ms / 1e3) / 1e9}
    if int(info["n_idx"]) == 0:  # entry-free plan (complete graph): no index stream at all
        if world == 1 and tm["launches"] <= 1:  # the whole K-step call was one launch
            roofline["kernel"] = ("single-launch trajectory kernel (k_persist_rk4, or k_small_dense for tiny graphs): "
                                  "avg_launch_ms is its time per RK4 stage = one RHS evaluation")
        roofline["note"] = ("entry-free plan: the SURVEY bytes are nominal -- the persistent trajectory kernel keeps "
                            "theta_n, acc, z and omega on chip for the whole kur_step, so per stage it moves only "
                            "its tile partials; it is bound by fp64 issue (sincos) and the per-stage grid "
                            "synchronisation, see profiles/r02/cfg2_k_persist_*")
    # the bound k_stage actually meets: the L1/shared-memory data pipe: one 16-byte z
    # read per hot entry from the staged window; nominal 128 B/clk/SM (B300_MICROARCH smem crossbar),
    # of which tools/mb_lds.cu reaches 99 % with slot ids in registers
    smem_peak = 128.0 * torch.cuda.get_device_properties(dev).multi_processor_count * (clk.max_mhz or 1965) * 1e6 / 1e9
    hot_alg, hot_issued = 16.0 * int(info["n_idx_hot"]), 16.0 * int(info["n_slots_hot"])
    smem_roofline = {"bound": "smem", "kernel": "k_remote + k_stage (overlapped pair)" if overlapped else "k_stage",
                     "unit": "GB/s", "peak": smem_peak,
                     "peak_source": "nominal 128 B/clk/SM x SMs x max SM clock",
                     "achieved": hot_alg / (kstage_ms / 1e3) / 1e9, "frac": hot_alg / (kstage_ms / 1e3) / 1e9 / smem_peak,
                     "issued_frac": hot_issued / (kstage_ms / 1e3) / 1e9 / smem_peak,
                     "bytes_per_launch": hot_alg, "bytes_formula": "16 B per hot (window-staged) entry"}

    # ---- SURVEY 8(d) protocol (i): back-to-back kur_rhs calls (z of the state, block sums, one
    # RHS; no RK epilogue), captured once in a CUDA graph and replayed (world 1 only)
    rhs_calls = None
    if world == 1 and not args.no_e2e:
        f_out = torch.empty_like(th)
        kur.rhs(g, th, om, K, out=f_out)
        torch.cuda.synchronize()
        ncall = 100 if inst.n >= (1 << 20) else 1000
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(10):
                kur.rhs(g, th, om, K, out=f_out)
        graph.replay()
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        for _ in range(ncall // 10):
            graph.replay()
        r1.record()
        torch.cuda.synchronize()
        r_ms = r0.elapsed_time(r1) / ncall
        rhs_calls = {"value": 1e3 / r_ms, "unit": UNIT, "calls": ncall, "ms_per_call": r_ms,
                     "path": "kur_rhs x 10 captured in a CUDA graph, replayed (prologue + [k_remote] + k_stage<RHS>)"}

    # ---- end to end through the public API with pinned host buffers
    e2e = None
    if not args.no_e2e:
        # the API works in internal order: the caller keeps its host state in that order.  The
        # state theta is the step's input and output and travels every step; omega (like the
        # graph) is a model parameter and stays resident on the device.
        th_hi = th.cpu().pin_memory()
        rt_h = torch.empty((2, 2), dtype=torch.float64).pin_memory()
        kur.step(g, th_hi, om, K, h, 1, 1)  # warm
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ne = max(3, min(args.steps, 20))
        ee0, ee1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ee0.record(stream)
        for _ in range(ne):
            rt = kur.step(g, th_hi, om, K, h, 1, 1)  # host theta in, 1 RK4 step, theta out (C ABI)
            rt_h.copy_(rt)
        ee1.record(stream)
        torch.cuda.synchronize()
        e_ms = ee0.elapsed_time(ee1) / ne
        if world > 1:
            t = torch.tensor([e_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        # value: global RHS evaluations per second (strong scaling); bytes: all ranks' copies
        e2e = {"value": 4.0 / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * inst.n,
               "d2h_bytes_per_step": 8 * inst.n + 32 * world, "ms_per_step": e_ms, "steps": ne,
               "path": "kur_step on the pinned HOST theta buffer: the library copies theta in, runs one RK4 step "
                       "and its last stage stores theta_{n+1} back through the buffer's device mapping; "
                       "then D2H of (r, psi); omega and the graph resident (model parameters)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_protocol(inst, args.config)

    ws = info["bytes_pool"] + 56 * inst.n
    l2_note = (f"inputs larger than L2 (index pool {info['bytes_pool'] / 1e9:.2f} GB + vectors vs 126 MB L2)"
               if ws > 126e6 else f"working set {ws / 1e6:.1f} MB is L2-resident and not flushed (a parity/"
               "latency case, not the bench line)")
    if rank == 0:
        out = {
            "metric": METRIC, "value": rhs_per_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": inst.name, "n": inst.n, "n_comm": inst.n_comm, "K": K, "h": h,
                       "nnz": int(info["nnz"]), "n_idx": int(info["n_idx"]), "seed": inst.seed,
                       "instance_sha256": inst.sha256()[:16], "l2": l2_note, "parallelism": f"communities x{world}",
                       "dense_threshold": args.dense_threshold,
                       "exchange": ("peer stores (fused)" if info["peer_exchange"] else "ncclAllGather")
                       if world > 1 else None},
            "rk4_steps_per_s": 1e3 / ms_per_step,
            "algorithmic_gbs": achieved,
            "roofline": roofline,
            "smem_roofline": smem_roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "rhs_calls": rhs_calls,
            # k_set_ctrl + every timed launch (prologue, k_remote, k_stage -- phase A and B at world > 1 --
            # or the one trajectory kernel) + k_unpack and k_finish per exchanged phase at world > 1
            "gpu_launches": 1 + tm["launches"] + (tm["stage_n"] if overlapped else 0)
                            + ((2 + int(info["peer_exchange"])) * (tm["prologue_n"] + tm["stage_n"]) if world > 1 else 0),
            "clocks": clk.result(),
            "host": dict(_host_info(), gen_s=gen_s, build_s=build_s),
            "plan": {k: info[k] for k in ("n_idx_hot", "n_idx_remote", "n_slots_hot", "n_slots_remote",
                                          "n_dense_blocks", "n_sparse_blocks", "n_tiles", "rows_per_tile",
                                          "bytes_per_rhs", "bytes_pool")},
            "csr_bytes_per_rhs": 4 * int(info["nnz"]),
            "r_final": r_final,
        }
        print(json.dumps(out), flush=True)
    g.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
