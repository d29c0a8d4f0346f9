#!/usr/bin/env python
"""Benchmark of the batched fp64 OCP-QP IPM (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--cfg C] [--path ocp|partial:<N1>|condense] [--batch B]
                    [--no-per-config]

A *step* is one complete batched solve (speed mode, tol 1e-8) of the
workload's whole batch.  BASELINE.json's metric names no configuration, so the
headline workload is the largest single-GPU configuration: BASELINE config 4
(256 random stage-varying QPs, nx=60, nu=20, N=100), solved directly by the
Riccati path.  Inputs are seeded synthetic data (generators.py; no dataset
exists for this path).  At N = 1 the same line carries a ``per_config`` block
with the other BASELINE configurations, each measured the same way: config 0
as single-QP latency, configs 1-3, and config 4's second way (partial
condensing to N2 = 20 blocks -> solve -> partial_expand).

* ``value``: whole-job solves/s with the batch resident in HBM, timed with CUDA
  events on the launching stream around each step (L2 flushed by a 512 MiB
  write between steps, outside the events); max over ranks for N > 1.
* ``e2e``: the same metric through the C ABI's host-buffer entry
  (ocpqp_solve_host): pinned host batch -> H2D -> solve -> D2H each step.
* ``roofline``: the fused solve kernel's algorithmic fp64 flops (SURVEY §8(d):
  sum over QPs of iterations x (F_fac + 2 F_sol)) / its event-timed duration,
  against the fp64 peak measured live by a DFMA microbenchmark (MEASURED_PEAKS
  has no fp64 entry); ``traffic`` = DRAM bytes per launch from the committed
  ncu capture of the same kernel source (null when the kernel sources changed
  since that capture: profiles/ncu_traffic.json records their hash).
* ``cpu_baseline``: the CPU oracle (oracle/, a C restatement of the reference
  pinned to its golden vectors) on all host cores over a bounded sample, with
  the parity of that sample against the GPU result.

``--impl reference`` times that CPU implementation alone on the same config
(rank 0 only under torchrun).  N > 1 runs independent replicas (the path
shards into independent QPs; no collective on the data path).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "batched OCP-QP IPM solves/s (fp64, 1 B200); Riccati % of FP64/HBM roofline"
HEADLINE_CFG = 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=HEADLINE_CFG)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=8.0,
                    help="target duration of the headline cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-config", action="store_true",
                    help="skip the per_config block (configs 0-3 and 4 via partial condensing)")
    ap.add_argument("--path", default="ocp",
                    help="ocp: the Riccati solve (headline); partial:<N1>: partial condensing "
                         "-> solve -> partial_expand (config 4's second way); condense: full "
                         "condensing -> dense-QP solve -> expand_solution (SURVEY 8(f) row 3)")
    ap.add_argument("--mode", default="speed",
                    choices=["speed", "sqrt", "balance", "robust", "speed_abs"],
                    help="IpmArg preset (sqrt = speed with the square-root Riccati variant); "
                         "the headline is speed")
    ap.add_argument("--tol", type=float, default=None,
                    help="exit tolerance (default 1e-8; 1e-6 for balance / robust, whose "
                         "lam_min = 1e-10 floors the reachable mu)")
    return ap.parse_args()


def make_arg(mode, tol):
    from dataclasses import replace

    from paper_2003_02547_b200.ipm import mode_preset

    if tol is None:
        tol = 1e-6 if mode in ("balance", "robust") else 1e-8
    if mode == "sqrt":
        return replace(mode_preset("speed").with_tol(tol), riccati_variant="square_root"), tol
    return mode_preset(mode).with_tol(tol), tol


def workload_name(cfg, B, mode="speed", tol=1e-8, path="ocp"):
    from paper_2003_02547_b200.generators import CONFIGS

    s = CONFIGS[cfg]
    if s.kind == "chain":
        desc = (f"{B} x spring chain M={s.masses} (nx={s.nx}, nu={s.nu}), N={s.N}, "
                f"seeded x0")
    else:
        desc = (f"{B} x random stage-varying OCP-QP (nx={s.nx}, nu={s.nu}, ng={s.ng}), "
                f"N={s.N}")
    mname = "speed mode" if mode == "speed" else (
        "speed mode, square-root Riccati" if mode == "sqrt" else f"{mode} mode")
    how = {"ocp": "direct Riccati solve",
           "condense": "full condensing + dense-QP solve + expand_solution"}.get(
        path, f"partial condensing N1={path.split(':')[-1]} + solve + partial_expand")
    return f"BASELINE config {cfg}: {desc}; {how}; {mname}, tol {tol:g}"


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during a region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0, interval_ms=20):
        self.index = index
        self.interval_ms = interval_ms
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", str(self.interval_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.05)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(names, parts[2:6]):
                if flag.lower() in ("active", "1", "yes"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "samples": len(sm), "reasons": sorted(reasons)}


def fp64_peak():
    import ctypes

    from paper_2003_02547_b200 import _native as nat

    L = nat.lib()
    L.ocpqp_fp64_peak.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
    a, b = ctypes.c_double(0), ctypes.c_double(0)
    rc = L.ocpqp_fp64_peak(ctypes.byref(a), ctypes.byref(b))
    if rc:
        return None, None
    return a.value, b.value


def kernel_source_hash():
    """Hash of the solve kernels' sources: ties an ncu capture to a build."""
    h = hashlib.sha256()
    csrc = ROOT / "paper_2003_02547_b200" / "csrc"
    for p in sorted(csrc.glob("*")):
        if p.suffix in (".cu", ".cuh", ".h"):
            h.update(p.name.encode())
            h.update(p.read_bytes())
    return h.hexdigest()[:16]


def ncu_traffic(key):
    """DRAM bytes per launch of the ncu capture recorded for `key`, if it was
    taken on the current kernel sources (else None with the reason)."""
    prof = ROOT / "profiles" / "ncu_traffic.json"
    try:
        tr = json.loads(prof.read_text()).get(key)
    except (ValueError, OSError):
        return None, "no ncu record"
    if not tr:
        return None, "no ncu record"
    if tr.get("src_hash") != kernel_source_hash():
        return None, f"ncu record {tr.get('source')} is from other kernel sources"
    return tr.get("dram_bytes_per_launch"), tr.get("source")


def host_info():
    cpu = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                cpu = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        gcc = subprocess.run(["gcc", "-dumpfullversion"], capture_output=True, text=True).stdout.strip()
    except OSError:
        gcc = "?"
    return {"cpu_model": cpu, "logical_cpus": os.cpu_count(), "numpy": np.__version__,
            "oracle_build": f"gcc {gcc} -O3 -march=x86-64-v3 (oracle/Makefile), pthreads"}


def rel_err_rows(a, r):
    return np.max(np.abs(a - r), axis=1) / np.maximum(1.0, np.max(np.abs(r), axis=1))


def run_cpu_oracle(batch, arg, seconds, max_qps=None, threads=None):
    """Oracle (C port) over all host cores; repeat the sample until `seconds`."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc  # test infrastructure; the cpu_baseline leg only

    orc.build()
    cores = threads or os.cpu_count() or 1
    sample = batch if max_qps is None or batch.B <= max_qps else batch.select(range(max_qps))
    t0 = time.perf_counter()
    out = orc.solve(sample, arg, nthreads=cores, trace=False)
    one = time.perf_counter() - t0
    reps, total = 1, one
    while total < seconds and reps < 1000:
        t0 = time.perf_counter()
        orc.solve(sample, arg, nthreads=cores, trace=False)
        total += time.perf_counter() - t0
        reps += 1
    cb = dict(value=sample.B * reps / total, unit="solves/s", cores=cores, kind="port",
              sample=f"{reps} x {sample.B} QPs of the workload ({total:.2f} s wall, "
                     f"{cores} threads, C restatement of the reference, oracle/)",
              **host_info())
    return cb, out, sample.B


def parity_block(out_np, ref, n):
    p = {"qps": n,
         "status_mismatch": int(np.sum(ref["status"] != out_np["status"][:n])),
         "iteration_mismatch": int(np.sum(ref["iters"] != out_np["iters"][:n]))}
    for k in ("y", "pi", "lam", "t"):
        e = rel_err_rows(out_np[k][:n], ref[k])
        p[f"max_rel_err_{k}"] = float(e.max())
        p[f"within_1e-8_{k}"] = int(np.sum(e <= 1e-8))
    d = np.abs(out_np["res"][:n] - ref["res"]) / np.maximum(1.0, np.abs(ref["res"]))
    p["max_res_norm_diff"] = float(np.nanmax(d)) if d.size else 0.0
    return p


class Ctx:
    def __init__(self, torch, device, stream, dist, world, rank):
        self.torch, self.device, self.stream = torch, device, stream
        self.dist, self.world, self.rank = dist, world, rank
        self.flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
        self.peak_dfma, self.peak_dmma = None, None

    def events(self, n):
        E = self.torch.cuda.Event
        return [(E(enable_timing=True), E(enable_timing=True)) for _ in range(n)]

    def max_over_ranks(self, v):
        if self.dist is None:
            return v
        tt = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(tt, op=self.dist.ReduceOp.MAX)
        return float(tt.item())


def bench_ocp(cx, cfg, B, arg, steps, warmup, *, e2e=True, cpu=True, cpu_seconds=5.0,
              cpu_max_qps=None, clocks=False):
    """The direct Riccati path on one config: value, roofline, e2e, cpu_baseline."""
    torch = cx.torch
    from paper_2003_02547_b200 import roofline as rf
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.ipm import team_supports
    from paper_2003_02547_b200.solver import get_plan, solve_ocp_qp_batch, solve_ocp_qp_host

    batch = make_batch(cfg, batch=B)
    dev = batch.to(cx.device)
    lay = batch.layout
    f64 = dict(dtype=torch.float64, device=cx.device)
    out = dict(y=torch.empty((B, lay.ny), **f64), pi=torch.empty((B, lay.ne), **f64),
               lam=torch.empty((B, lay.nc), **f64), t=torch.empty((B, lay.nc), **f64),
               status=torch.empty(B, dtype=torch.int32, device=cx.device),
               iters=torch.empty(B, dtype=torch.int32, device=cx.device),
               res=torch.empty((B, 5), **f64), flops=torch.empty(B, dtype=torch.int64, device=cx.device),
               trace=None)
    stream = cx.stream

    def step():
        return solve_ocp_qp_batch(dev, arg, trace=False, out=out, stream=stream)

    # warm-up: at least W steps and ~0.3 s so clocks settle
    t_end = time.perf_counter() + 0.3
    w = 0
    while w < warmup or time.perf_counter() < t_end:
        step()
        w += 1
        if w % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    plan_info = get_plan(dev).info()
    if plan_info.get("kernel") == "team" and not team_supports(
            arg, int(batch.dim.nx[0]) + int(batch.dim.nu[0]), int(batch.dim.nx[0])):
        plan_info["kernel"] = "generic"   # square-root / robust run on k_ipm_solve
    evs = cx.events(steps)
    sampler = ClockSampler(index=cx.device.index or 0) if clocks else None
    if cx.dist is not None:
        cx.dist.barrier()
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.05)
    for e0, e1 in evs:
        cx.flush.zero_()
        e0.record(stream)
        step()
        e1.record(stream)
    torch.cuda.synchronize()
    clk = sampler.stop() if sampler else None
    if cx.dist is not None:
        cx.dist.barrier()
    times = np.array([e0.elapsed_time(e1) for e0, e1 in evs])  # ms
    t_step = cx.max_over_ranks(float(times.mean()))
    value = cx.world * B / (t_step * 1e-3)

    o = {k: out[k].cpu().numpy() for k in ("y", "pi", "lam", "t", "status", "iters", "res")}
    iters = o["iters"].astype(np.int64)
    ric = rf.riccati_flops(batch.dim)
    achieved = float(iters.sum()) * ric / (t_step * 1e-3) / 1e12
    kname = {"row": "k_row_solve", "team": "k_fast_solve"}.get(plan_info.get("kernel"), "k_ipm_solve")
    traffic, tsrc = ncu_traffic(f"cfg{cfg}")
    roof = {"bound": "tensor", "pipe": "fp64 (DFMA / DMMA)", "achieved": achieved,
            "peak": cx.peak_dfma, "unit": "TFLOP/s",
            "frac": achieved / cx.peak_dfma if cx.peak_dfma else None,
            "traffic": traffic, "traffic_source": tsrc, "kernel": kname,
            "work": f"sum over QPs of iterations x (F_fac + 2 F_sol) = {int(iters.sum())} x {ric} "
                    f"flops (SURVEY §8(d)); one solve launch per step",
            "peak_source": ("measured live: DFMA microbenchmark (ocpqp_fp64_peak), "
                            f"DMMA m8n8k4 {cx.peak_dmma:.1f} TFLOP/s") if cx.peak_dmma else "n/a",
            "algorithmic_bytes_per_launch": float(iters.sum()) * rf.stream_bytes(batch.dim, lay),
            "hbm_peak_gbs": 6549.4}
    roof["hbm_frac_of_algorithmic_bytes"] = (roof["algorithmic_bytes_per_launch"] / (t_step * 1e-3)
                                             / 1e9 / roof["hbm_peak_gbs"])
    # Riccati share of the kernel time (the metric's "Riccati % of roofline"):
    # one extra, untimed solve with the kernel's clock64 phase counters; the
    # factor recursion (T1, G, Cholesky, K, P) and the backward / forward
    # sweeps are the Riccati phases, the rest are the IPM vector passes
    if plan_info.get("kernel") == "team":
        try:
            dbg = torch.zeros((B, 24), dtype=torch.int64, device=cx.device)
            solve_ocp_qp_batch(dev, arg, trace=False, phase_debug=dbg, stream=stream)
            torch.cuda.synchronize()
            solve_ocp_qp_batch(dev, arg, trace=False, stream=stream)  # instrumentation off
            ph = dbg.cpu().numpy().astype(np.float64)
            r_ph = ph[:, [8, 9, 10, 11, 12, 14, 15]].sum()
            tot = ph[:, 5].sum()
            if tot > 0 and r_ph > 0:
                share = float(r_ph / tot)
                roof["riccati"] = {
                    "share_of_kernel_time": share,
                    "achieved": achieved / share, "frac": roof["frac"] / share if roof["frac"] else None,
                    "phases": "factor recursion (T1, G, Cholesky, K, P) + backward/forward sweeps; "
                              "clock64 phase counters summed over QPs, one extra untimed solve"}
        except Exception as exc:  # diagnostics only
            roof["riccati"] = {"error": str(exc)[:120]}
    # our kernels per solve (ocpqp_solve): the team kernel path launches the
    # stage-invariance check, the [B A] pack and the solve, plus the generic
    # kernel over the escape list in balance mode; the generic path one kernel
    if plan_info.get("kernel") == "team":
        launches = 3 + (1 if arg.use_qr_fallback else 0)
    else:
        launches = 1
    res = {"value": value, "unit": "solves/s", "ms_per_step": t_step, "steps": steps, "warmup": w,
           "roofline": roof, "gpu_launches": steps * launches, "plan": plan_info,
           "iterations": {"min": int(iters.min()), "mean": float(iters.mean()),
                          "max": int(iters.max())},
           "status_counts": {str(int(k)): int(v) for k, v in
                             zip(*np.unique(o["status"], return_counts=True))},
           "step_ms": {"min": float(times.min()), "median": float(np.median(times)),
                       "max": float(times.max())}}
    if clk is not None:
        res["clocks"] = clk
    if plan_info.get("kernel") == "team" and cx.world == 1 and cfg == 4:
        # Not part of `value`: the same batch with the plan's opt-in dispatch hint
        # (ocpqp_plan_dispatch_hint: QPs handed out by the PREVIOUS solve's iteration
        # counts, the slowest to the CTAs alone on their SM).  It needs a previous solve
        # of a similar batch (closed-loop MPC); here that is the identical batch, so the
        # number shows what the launch's tail costs, not the one-shot throughput.
        plan = get_plan(dev)
        plan.dispatch_hint(True)
        try:
            for _ in range(3):
                step()
            hev = cx.events(5)
            for e0, e1 in hev:
                cx.flush.zero_()
                e0.record(stream)
                step()
                e1.record(stream)
            torch.cuda.synchronize()
            th = float(np.mean([e0.elapsed_time(e1) for e0, e1 in hev]))
            same = bool(np.array_equal(out["iters"].cpu().numpy(), o["iters"])) and all(
                bool(np.array_equal(out[k].cpu().numpy(), o[k])) for k in ("y", "pi", "lam", "t"))
            res["dispatch_hint"] = {
                "value": B / (th * 1e-3), "unit": "solves/s", "ms_per_step": th, "steps": 5,
                "identical_results": same,
                "note": "opt-in, off in `value`: QP order from the plan's previous solve of the "
                        "same batch (slowest QPs to the CTAs alone on their SM)"}
        finally:
            plan.dispatch_hint(False)
            step()
            torch.cuda.synchronize()
    if e2e:
        hb = batch.pin_memory()
        hout = dict(y=torch.empty((B, lay.ny), dtype=torch.float64).pin_memory(),
                    pi=torch.empty((B, lay.ne), dtype=torch.float64).pin_memory(),
                    lam=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
                    t=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
                    status=torch.empty(B, dtype=torch.int32).pin_memory(),
                    iters=torch.empty(B, dtype=torch.int32).pin_memory(),
                    res=torch.empty((B, 5), dtype=torch.float64).pin_memory(),
                    flops=torch.empty(B, dtype=torch.int64).pin_memory(), trace=None)
        for _ in range(2):
            solve_ocp_qp_host(hb, arg, out=hout, stream=stream)
        et = []
        ksteps = max(3, steps // 4)
        for _ in range(ksteps):
            cx.flush.zero_()
            e0, e1 = cx.events(1)[0]
            e0.record(stream)
            solve_ocp_qp_host(hb, arg, out=hout, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            et.append(e0.elapsed_time(e1))
        te = cx.max_over_ranks(float(np.mean(et)))
        h2d = sum(int(v.numel()) * 8 for v in hb.fields.values())
        d2h = sum(int(hout[k].numel()) * hout[k].element_size()
                  for k in ("y", "pi", "lam", "t", "status", "iters", "res", "flops"))
        res["e2e"] = {"value": cx.world * B / (te * 1e-3), "unit": "solves/s",
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                      "ms_per_step": te, "steps": ksteps,
                      "iterations_match_device_path": bool(np.array_equal(hout["iters"].numpy(), iters))}
    if cpu and cx.rank == 0 and cx.world == 1:
        cb, ref, n = run_cpu_oracle(batch, arg, seconds=cpu_seconds, max_qps=cpu_max_qps)
        res["cpu_baseline"] = cb
        res["parity_vs_oracle"] = parity_block(o, ref, n)
    return res


def bench_latency(cx, cfg, arg, steps):
    """Single-QP latency (BASELINE config 0): one solve per step, B = 1."""
    torch = cx.torch
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.solver import solve_ocp_qp_batch, solve_ocp_qp_host

    r = bench_ocp(cx, cfg, 1, arg, steps, 20, e2e=False, cpu=False)
    batch = make_batch(cfg, batch=1)
    # e2e: the reference-facing host call, host buffers in and out
    hb = batch.pin_memory()
    for _ in range(5):
        solve_ocp_qp_host(hb, arg, stream=cx.stream)
    torch.cuda.synchronize()
    et = []
    for _ in range(steps):
        e0, e1 = cx.events(1)[0]
        e0.record(cx.stream)
        rep = solve_ocp_qp_host(hb, arg, stream=cx.stream)
        e1.record(cx.stream)
        torch.cuda.synchronize()
        et.append(e0.elapsed_time(e1))
    te = float(np.median(et))
    r["latency_ms"] = r["ms_per_step"]
    r["e2e"] = {"value": 1e3 / te, "unit": "solves/s", "latency_ms": te,
                "h2d_bytes_per_step": sum(int(v.numel()) * 8 for v in hb.fields.values()),
                "d2h_bytes_per_step": int(sum(np.asarray(getattr(rep, k)).nbytes
                                              for k in ("y", "pi", "lam", "t"))) + 4 + 4 + 40 + 8,
                "steps": steps}
    if cx.rank == 0:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle as orc  # cpu_baseline leg only

        orc.build()
        t0 = time.perf_counter()
        n = 0
        while time.perf_counter() - t0 < 2.0:
            ref = orc.solve(batch, arg, nthreads=1, trace=False)
            n += 1
        lat = (time.perf_counter() - t0) / n
        r["cpu_baseline"] = {"value": 1.0 / lat, "unit": "solves/s", "latency_ms": lat * 1e3,
                             "cores": 1, "kind": "port",
                             "sample": f"{n} single-QP solves on one thread (C restatement)",
                             **host_info()}
        g = solve_ocp_qp_batch(batch.to(cx.device), arg, trace=False)
        o = {k: getattr(g, k).cpu().numpy() for k in ("y", "pi", "lam", "t", "res")}
        o["status"], o["iters"] = g.status_code.cpu().numpy(), g.iterations.cpu().numpy()
        r["parity_vs_oracle"] = parity_block(o, ref, 1)
    return r


def bench_condense(cx, cfg, B, arg, path, steps, warmup, *, e2e=True, cpu=True, clocks=False):
    """Condensing paths: partial:<N1> (config 4's second way) or condense.

    value: QPs/s through the three device stages (condense -> solve -> expand),
    inputs resident; roofline of the dominant kernel (the condensed solve):
    the reference's own counted flops of that solve (identical to ours) over
    its event-timed duration; e2e: the same from pinned host buffers (one H2D
    of the source batch per step), the expanded (y, pi, lam, t) and status /
    iterations read back.  cpu_baseline: the oracle's own path (numpy
    restatement of condensing + C solve + numpy expansion) on a sample, whose
    expanded solution is compared with the GPU's.
    """
    torch = cx.torch
    from paper_2003_02547_b200.condensing import (condense_batch, expand_batch,
                                                  partial_condense_batch, partial_expand_batch)
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.solver import get_plan, solve_ocp_qp_batch

    full = path == "condense"
    N1 = None if full else int(path.split(":", 1)[1])
    batch = make_batch(cfg, batch=B)
    dev = batch.to(cx.device)
    stream = cx.stream

    def step(src, ev=None):
        cb, cmap = condense_batch(src) if full else partial_condense_batch(src, N1)
        if ev is not None:
            ev[0].record(stream)
        rep = solve_ocp_qp_batch(cb, arg, trace=False, stream=stream)
        if ev is not None:
            ev[1].record(stream)
        ex = expand_batch if full else partial_expand_batch
        return cb, rep, ex(rep, cmap, src)

    w = 0
    t_end = time.perf_counter() + 0.3
    while w < warmup or time.perf_counter() < t_end:
        step(dev)
        w += 1
    torch.cuda.synchronize()
    evs = [(a, b, cx.events(1)[0]) for a, b in cx.events(steps)]
    sampler = ClockSampler(index=cx.device.index or 0) if clocks else None
    torch.cuda.synchronize()
    if sampler:
        sampler.start()
        time.sleep(0.05)
    for e0, e1, ek in evs:
        cx.flush.zero_()
        e0.record(stream)
        cb, rep, expd = step(dev, ek)
        e1.record(stream)
    torch.cuda.synchronize()
    clk = sampler.stop() if sampler else None
    times = np.array([e0.elapsed_time(e1) for e0, e1, _ in evs])
    ktimes = np.array([ek[0].elapsed_time(ek[1]) for _, _, ek in evs])
    t_step = cx.max_over_ranks(float(times.mean()))
    t_k = float(ktimes.mean())
    flops = float(rep.flops.sum().item())
    iters = rep.iterations.cpu().numpy()
    status = rep.status_code.cpu().numpy()
    achieved = flops / (t_k * 1e-3) / 1e12
    plan_info = get_plan(cb).info()
    traffic, tsrc = ncu_traffic(f"cfg{cfg}-{path}")
    res = {"value": cx.world * B / (t_step * 1e-3), "unit": "solves/s", "ms_per_step": t_step,
           "steps": steps, "warmup": w, "path": path,
           "roofline": {"bound": "tensor", "pipe": "fp64 (DFMA / DMMA)", "achieved": achieved,
                        "peak": cx.peak_dfma, "unit": "TFLOP/s",
                        "frac": achieved / cx.peak_dfma if cx.peak_dfma else None,
                        "traffic": traffic, "traffic_source": tsrc,
                        "kernel": ("k_ipm_solve (dense N = 0 form)" if full else
                                   f"{plan_info.get('kernel')} kernel on the condensed QPs"),
                        "work": f"reference-counted flops of the condensed solves = {flops:.4g} "
                                f"per step over the solve kernel's {t_k:.3f} ms",
                        "kernel_share_of_step": t_k / t_step},
           "gpu_launches": steps * 3, "plan": plan_info,
           "stage_ms": {"solve": t_k, "condense_plus_expand": t_step - t_k},
           "condensed_dims": {"N": int(cb.dim.N), "nu": [int(v) for v in cb.dim.nu[:2]],
                              "nb": [int(v) for v in cb.dim.nb[:2]],
                              "ng": [int(v) for v in cb.dim.ng[:2]]},
           "iterations": {"min": int(iters.min()), "mean": float(iters.mean()),
                          "max": int(iters.max())},
           "status_counts": {str(int(k)): int(v) for k, v in zip(*np.unique(status, return_counts=True))}}
    if clk is not None:
        res["clocks"] = clk
    if e2e:
        hb = batch.pin_memory()
        et = []
        h2d = sum(int(v.numel()) * 8 for v in hb.fields.values())
        for i in range(max(3, steps // 4) + 2):
            cx.flush.zero_()
            e0, e1 = cx.events(1)[0]
            e0.record(stream)
            src = hb.to(cx.device)        # the step's one host -> device copy
            _, r2, (y, pi, lam, t) = step(src)
            outs = [x.to("cpu", non_blocking=True) for x in (y, pi, lam, t, r2.status_code,
                                                            r2.iterations)]
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                et.append(e0.elapsed_time(e1))
        te = cx.max_over_ranks(float(np.mean(et)))
        res["e2e"] = {"value": cx.world * B / (te * 1e-3), "unit": "solves/s",
                      "h2d_bytes_per_step": h2d,
                      "d2h_bytes_per_step": sum(int(x.numel()) * x.element_size() for x in outs),
                      "ms_per_step": te, "steps": len(et)}
    if cpu and cx.rank == 0 and cx.world == 1:
        sys.path.insert(0, str(ROOT / "oracle"))
        import condense_oracle as co  # test infrastructure; the cpu_baseline leg only
        import oracle as orc

        from paper_2003_02547_b200 import OcpQpBatch, dense_to_ocp
        from paper_2003_02547_b200.dense import DenseQp
        from paper_2003_02547_b200.layout import OcpLayout

        orc.build()
        cores = os.cpu_count() or 1
        n = min(B, 64) if full else max(2, min(B, cores))
        qps = [batch.qp(i) for i in range(n)]
        t0 = time.perf_counter()
        exp = []
        if not full:
            cq = [co.partial_condensed_qp(q, N1) for q in qps]
            ob = OcpQpBatch.from_qps([c[0] for c in cq])
            ref = orc.solve(ob, arg, nthreads=cores, trace=False)
            lay2 = OcpLayout(ob.dim)
            for i, q in enumerate(qps):
                exp.append(co.partial_expand(q, cq[i][1], dict(
                    layout=lay2, y=ref["y"][i], pi=ref["pi"][i], lam=ref["lam"][i], t=ref["t"][i])))
        else:
            dqs, maps = [], []
            for q in qps:
                dd, m = co.full_condense(q)
                dq = DenseQp(len(dd["g"]), 0, len(dd["idxb"]), len(dd["lg"]), 0)
                for f in ("H", "g", "idxb", "lb", "ub", "C", "lg", "ug", "maskl", "masku"):
                    dq.set_field(f, dd[f])
                dqs.append(dense_to_ocp(dq))
                maps.append(m)
            ref = orc.solve(OcpQpBatch.from_qps(dqs), arg, nthreads=cores, trace=False)
            for i, q in enumerate(qps):
                exp.append(co.full_expand(q, maps[i], ref["y"][i], ref["lam"][i], ref["t"][i]))
        tc = time.perf_counter() - t0
        res["cpu_baseline"] = {"value": n / tc, "unit": "solves/s", "cores": cores, "kind": "port",
                               "sample": f"{n} QPs of the workload: numpy "
                                         f"{'condense' if full else 'partial_condense'} + C-oracle "
                                         f"solve ({cores} threads) + numpy expand, {tc:.2f} s",
                               **host_info()}
        par = {"qps": n, "status_mismatch": int(np.sum(ref["status"] != status[:n])),
               "iteration_mismatch": int(np.sum(ref["iters"] != iters[:n]))}
        for j, k in enumerate(("y", "pi", "lam", "t")):
            if full and k == "pi":
                continue
            g = expd[j].cpu().numpy()[:n]
            r = np.stack([e[j if not full else {"y": 0, "lam": 1, "t": 2}[k]] for e in exp])
            e = rel_err_rows(g, r)
            par[f"max_rel_err_{k}"] = float(e.max())
            par[f"within_1e-8_{k}"] = int(np.sum(e <= 1e-8))
        res["parity_vs_oracle"] = par
    return res


def reference_arm(a, arg, config, B):
    """--impl reference: the reference's CPU implementation of the path (the C
    restatement; the Python reference cannot travel to the GPU box) on all
    host threads, each step a bounded sample of the same workload."""
    from paper_2003_02547_b200.generators import CONFIGS, make_batch

    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc  # the reference arm: the one other place bench runs oracle/

    orc.build()
    cores = os.cpu_count() or 1
    chain = CONFIGS[a.cfg].kind == "chain"
    nq = B if chain else min(B, max(cores, 8))
    batch = make_batch(a.cfg, batch=nq)
    for _ in range(max(0, a.warmup)):
        orc.solve(batch, arg, nthreads=cores, trace=False)
    samples = []
    for _ in range(max(1, a.steps)):
        t0 = time.perf_counter()
        orc.solve(batch, arg, nthreads=cores, trace=False)
        samples.append(time.perf_counter() - t0)
        if sum(samples) > 90.0:
            break
    t = float(np.mean(samples))
    value = nq / t
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": a.gpus,
            "steps": len(samples), "warmup": a.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded generators, BASELINE configs)",
            "config": config, "impl": "reference",
            "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cores, "kind": "port",
                             "sample": f"{nq} QPs of the workload per step, {cores} threads "
                                       f"(C restatement of the reference, oracle/)",
                             **host_info()},
            "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2003_02547_b200.generators import CONFIGS

    arg, tol = make_arg(a.mode, a.tol)
    B = a.batch or CONFIGS[a.cfg].batch
    config = {"workload": workload_name(a.cfg, B, a.mode, tol, a.path), "batch_per_gpu": B,
              "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
              "l2": "flushed between steps (512 MiB write outside the timed events)"}
    if a.impl == "reference":
        if rank == 0:
            reference_arm(a, arg, config, B)
        return

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    cx = Ctx(torch, device, torch.cuda.current_stream(device), dist, world, rank)
    cx.peak_dfma, cx.peak_dmma = fp64_peak()

    cpu_max = None if CONFIGS[a.cfg].kind == "chain" else max(8, min(B, os.cpu_count() or 8))
    if a.path == "ocp":
        r = bench_ocp(cx, a.cfg, B, arg, a.steps, a.warmup, e2e=not a.no_e2e,
                      cpu=not a.no_cpu_baseline, cpu_seconds=a.cpu_seconds, cpu_max_qps=cpu_max,
                      clocks=True)
    else:
        r = bench_condense(cx, a.cfg, B, arg, a.path, a.steps, a.warmup, e2e=not a.no_e2e,
                           cpu=not a.no_cpu_baseline, clocks=True)
    line = {"metric": METRIC, "value": r.pop("value"), "unit": r.pop("unit"), "n_gpus": world,
            "steps": a.steps, "warmup": r.pop("warmup"), "ms_per_step": r.pop("ms_per_step"),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, BASELINE configs)", "config": config}
    r.pop("steps", None)
    line.update(r)
    if world == 1 and not a.no_per_config and a.mode == "speed" and a.path == "ocp" and a.batch is None:
        per = {}
        per["0"] = dict(workload=workload_name(0, 1, a.mode, tol),
                        **bench_latency(cx, 0, arg, steps=50))
        for c in (1, 2, 3):
            if c == a.cfg:
                continue
            Bc = CONFIGS[c].batch
            per[str(c)] = dict(workload=workload_name(c, Bc, a.mode, tol),
                               **bench_ocp(cx, c, Bc, arg, 10 if c == 1 else 5, 3, cpu_seconds=3.0,
                                           cpu_max_qps=None if c == 1 else max(16, os.cpu_count() or 16)))
        if a.cfg == 4:
            per["4-partial"] = dict(workload=workload_name(4, 256, a.mode, tol, "partial:5"),
                                    **bench_condense(cx, 4, 256, arg, "partial:5", 3, 2))
        line["per_config"] = per
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
