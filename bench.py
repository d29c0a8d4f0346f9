#!/usr/bin/env python
"""Benchmark of the batched fp64 OCP-QP IPM (driver contract, one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--cfg C] [--batch B]

A *step* is one complete batched solve (speed mode, tol 1e-8) of the
workload's whole batch.  Default workload: BASELINE config 1 (1024 QPs, 4-mass
spring chain, nx=8, nu=3, N=15), the configuration BASELINE.json's metric is
quoted on; inputs are seeded synthetic data (generators.py).

* ``value``: whole-job solves/s with the batch resident in HBM, timed with CUDA
  events on the launching stream around each step (L2 flushed by a 512 MiB
  write between steps, outside the events); max over ranks for N > 1.
* ``e2e``: the same metric through the C ABI's host-buffer entry
  (ocpqp_solve_host): pinned host batch -> H2D -> solve -> D2H each step.
* ``roofline``: the fused solve kernel's algorithmic fp64 flops (SURVEY §8(d):
  sum over QPs of iterations x (F_fac + 2 F_sol)) / its event-timed duration,
  against the fp64 peak measured live by a DFMA microbenchmark (MEASURED_PEAKS
  has no fp64 entry).
* ``cpu_baseline``: the CPU oracle (oracle/, a C restatement of the reference
  pinned to its golden vectors) on all host cores over a bounded sample.

``--impl reference`` times that CPU implementation alone on the same config
(rank 0 only under torchrun).  N > 1 runs independent replicas (the path
shards into independent QPs; no collective on the data path).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "batched OCP-QP IPM solves/s (fp64, 1 B200); Riccati % of FP64/HBM roofline"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cfg", type=int, default=1)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--cpu-seconds", type=float, default=3.0,
                    help="target duration of the cpu_baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
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


def workload_name(cfg, B, mode="speed", tol=1e-8):
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
    return f"BASELINE config {cfg}: {desc}; {mname}, tol {tol:g}"


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


def run_cpu_oracle(batch, arg, seconds, max_qps=None):
    """Oracle (C port) over all host cores; repeat the sample until `seconds`."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle as orc  # test infrastructure; the cpu_baseline leg only

    orc.build()
    cores = os.cpu_count() or 1
    sample = batch if max_qps is None or batch.B <= max_qps else batch.select(range(max_qps))
    t0 = time.perf_counter()
    out = orc.solve(sample, arg, nthreads=cores, trace=False)
    one = time.perf_counter() - t0
    reps = 1
    total = one
    while total < seconds and reps < 1000:
        t0 = time.perf_counter()
        orc.solve(sample, arg, nthreads=cores, trace=False)
        total += time.perf_counter() - t0
        reps += 1
    return dict(value=sample.B * reps / total, unit="solves/s", cores=cores, kind="port",
                sample=f"{reps} x {sample.B} QPs of the workload ({total:.2f} s wall, "
                       f"{cores} threads, C restatement of the reference, oracle/)",
                per_step_s=total / reps, qps=sample.B), out


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2003_02547_b200.generators import CONFIGS, make_batch

    arg, tol = make_arg(a.mode, a.tol)
    B = a.batch or CONFIGS[a.cfg].batch
    config = {"workload": workload_name(a.cfg, B, a.mode, tol), "batch_per_gpu": B,
              "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
              "l2": "flushed between steps (512 MiB write outside the timed events)"}

    if a.impl == "reference":
        if rank != 0:
            return
        batch = make_batch(a.cfg, batch=B)
        samples = []
        for _ in range(max(0, a.warmup)):
            pass
        max_qps = None if CONFIGS[a.cfg].kind == "chain" else max(8, min(B, 64))
        cb, _ = run_cpu_oracle(batch, arg, seconds=0.0, max_qps=max_qps)
        for _ in range(max(1, a.steps)):
            c, _ = run_cpu_oracle(batch, arg, seconds=0.0, max_qps=max_qps)
            samples.append(c["per_step_s"])
            if sum(samples) > 60.0:
                break
        t = float(np.mean(samples))
        value = cb["qps"] / t
        line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
                "steps": len(samples), "warmup": a.warmup, "ms_per_step": t * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded generators, BASELINE configs)",
                "config": config, "impl": "reference",
                "cpu_baseline": {"value": value, "unit": "solves/s", "cores": cb["cores"],
                                 "kind": "port",
                                 "sample": f"{cb['qps']} QPs per step, {cb['cores']} threads"},
                "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if a.path == "condense" or a.path.startswith("partial:"):
        return main_condense(a, arg, B, config, rank, world, local)
    if a.path != "ocp":
        raise SystemExit(f"unknown --path {a.path}")

    import torch

    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)

    from paper_2003_02547_b200 import roofline as rf
    from paper_2003_02547_b200.solver import get_plan, solve_ocp_qp_batch, solve_ocp_qp_host

    batch = make_batch(a.cfg, batch=B)
    dev = batch.to(device)
    lay = batch.layout
    f64 = dict(dtype=torch.float64, device=device)
    out = dict(y=torch.empty((B, lay.ny), **f64), pi=torch.empty((B, lay.ne), **f64),
               lam=torch.empty((B, lay.nc), **f64), t=torch.empty((B, lay.nc), **f64),
               status=torch.empty(B, dtype=torch.int32, device=device),
               iters=torch.empty(B, dtype=torch.int32, device=device),
               res=torch.empty((B, 5), **f64), flops=torch.empty(B, dtype=torch.int64, device=device),
               trace=None)
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)

    def step():
        return solve_ocp_qp_batch(dev, arg, trace=False, out=out, stream=stream)

    # warm-up: at least W steps and ~0.5 s so clocks settle
    t_end = time.perf_counter() + 0.5
    w = 0
    while w < a.warmup or time.perf_counter() < t_end:
        step()
        w += 1
        if w % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    plan_info = get_plan(dev).info()
    from paper_2003_02547_b200.ipm import team_supports

    if plan_info.get("kernel") == "team" and not team_supports(
            arg, int(batch.dim.nx[0]) + int(batch.dim.nu[0])):
        plan_info["kernel"] = "generic"   # square-root / robust run on k_ipm_solve

    peak_dfma, peak_dmma = fp64_peak()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(a.steps)]
    sampler = ClockSampler(index=local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.05)
    for e0, e1 in evs:
        flush.zero_()
        e0.record(stream)
        step()
        e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if dist is not None:
        dist.barrier()
    times = np.array([e0.elapsed_time(e1) for e0, e1 in evs])  # ms
    t_step = float(times.mean())
    if dist is not None:
        tt = torch.tensor([t_step], dtype=torch.float64, device=device)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    value = world * B / (t_step * 1e-3)

    iters = out["iters"].cpu().numpy().astype(np.int64)
    status = out["status"].cpu().numpy()
    ric = rf.riccati_flops(batch.dim)
    alg_flops = float(iters.sum()) * ric
    achieved = alg_flops / (t_step * 1e-3) / 1e12
    # compute-bound roofline of the FP64 pipes: MEASURED_PEAKS.json and the
    # profiling guide carry no FP64 figure, so the peak is measured live on
    # this GPU (DFMA chain microbenchmark; the FP64 tensor-core DMMA path
    # measures the same).  "tensor" = compute-bound in the contract's terms.
    roof = {"bound": "tensor", "pipe": "fp64 (DFMA / DMMA)", "achieved": achieved, "peak": peak_dfma,
            "unit": "TFLOP/s",
            "frac": achieved / peak_dfma if peak_dfma else None, "traffic": None,
            "kernel": {"row": "k_row_solve", "team": "k_fast_solve"}.get(plan_info.get("kernel"), "k_ipm_solve"),
            "work": f"sum over QPs of iterations x (F_fac + 2 F_sol) = {iters.sum()} x {ric} flops "
                    f"(SURVEY §8(d)); one launch per step",
            "peak_source": "measured live: DFMA microbenchmark (ocpqp_fp64_peak), "
                           f"DMMA m8n8k4 {peak_dmma:.1f} TFLOP/s" if peak_dmma else "n/a",
            "stream_bytes_per_qp_iter": rf.stream_bytes(batch.dim, lay)}
    # Riccati share of the kernel time (the metric's "Riccati % of roofline"):
    # one extra, untimed solve with the kernel's clock64 phase counters; the
    # factor recursion (T1, G, Cholesky, K, P) and the backward / forward
    # sweeps are the Riccati phases, the rest are the IPM vector passes
    if plan_info.get("kernel") == "team":
        try:
            dbg = torch.zeros((B, 16), dtype=torch.int64, device="cuda")
            solve_ocp_qp_batch(dev, arg, trace=False, phase_debug=dbg, stream=stream)
            torch.cuda.synchronize()
            solve_ocp_qp_batch(dev, arg, trace=False, stream=stream)  # instrumentation off
            ph = dbg.cpu().numpy().astype(np.float64)
            ric = ph[:, [8, 9, 10, 11, 12, 14, 15]].sum()
            tot = ph[:, 5].sum()
            if tot > 0 and ric > 0:
                share = float(ric / tot)
                roof["riccati"] = {
                    "share_of_kernel_time": share,
                    "achieved": achieved / share, "frac": roof["frac"] / share if roof["frac"] else None,
                    "phases": "factor recursion (T1, G, Cholesky, K, P) + backward/forward sweeps; "
                              "clock64 phase counters summed over QPs, one extra untimed solve"}
        except Exception as exc:  # diagnostics only
            roof["riccati"] = {"error": str(exc)[:120]}
    prof = ROOT / "profiles" / "ncu_traffic.json"
    if prof.exists():
        try:
            tr = json.loads(prof.read_text()).get(str(a.cfg))
            if tr:
                roof["traffic"] = tr.get("dram_bytes_per_launch")
        except (ValueError, OSError):
            pass

    # our kernels per solve (ocpqp_solve): the team kernel path launches the
    # stage-invariance check, the [B A] pack and the solve, plus the generic
    # kernel over the escape list in balance mode; the generic path one kernel
    if plan_info.get("kernel") == "team":
        launches_per_solve = 3 + (1 if arg.use_qr_fallback else 0)
    else:
        launches_per_solve = 1
    line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": a.steps, "warmup": w, "ms_per_step": t_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, BASELINE configs)", "config": config,
            "roofline": roof, "clocks": clocks, "gpu_launches": a.steps * launches_per_solve,
            "plan": plan_info,
            "iterations": {"min": int(iters.min()), "mean": float(iters.mean()),
                           "max": int(iters.max())},
            "status_counts": {str(int(k)): int(v) for k, v in zip(*np.unique(status, return_counts=True))},
            "step_ms": {"min": float(times.min()), "median": float(np.median(times)),
                        "max": float(times.max())}}

    # ---- end to end through the host-buffer C ABI entry ----
    if not a.no_e2e:
        hb = batch.pin_memory()
        hout = dict(y=torch.empty((B, lay.ny), dtype=torch.float64).pin_memory(),
                    pi=torch.empty((B, lay.ne), dtype=torch.float64).pin_memory(),
                    lam=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
                    t=torch.empty((B, lay.nc), dtype=torch.float64).pin_memory(),
                    status=torch.empty(B, dtype=torch.int32).pin_memory(),
                    iters=torch.empty(B, dtype=torch.int32).pin_memory(),
                    res=torch.empty((B, 5), dtype=torch.float64).pin_memory(),
                    flops=torch.empty(B, dtype=torch.int64).pin_memory(), trace=None)
        for _ in range(3):
            solve_ocp_qp_host(hb, arg, out=hout, stream=stream)
        et = []
        ksteps = max(5, a.steps // 4)
        for _ in range(ksteps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            solve_ocp_qp_host(hb, arg, out=hout, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            et.append(e0.elapsed_time(e1))
        te = float(np.mean(et))
        h2d = sum(int(v.numel()) * 8 for v in hb.fields.values())
        d2h = sum(int(hout[k].numel()) * hout[k].element_size()
                  for k in ("y", "pi", "lam", "t", "status", "iters", "res", "flops"))
        e2e_iters = hout["iters"].numpy()
        line["e2e"] = {"value": world * B / (te * 1e-3), "unit": "solves/s",
                       "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "ms_per_step": te, "steps": ksteps,
                       "iterations_match_device_path": bool(np.array_equal(e2e_iters, iters))}

    # ---- CPU baseline (rank 0, N == 1) ----
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        max_qps = None if CONFIGS[a.cfg].kind == "chain" else 64
        cb, ref = run_cpu_oracle(batch, arg, seconds=a.cpu_seconds, max_qps=max_qps)
        n = ref["iters"].shape[0]
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        line["parity_vs_oracle"] = {
            "qps": n,
            "status_mismatch": int(np.sum(ref["status"] != status[:n])),
            "iteration_mismatch": int(np.sum(ref["iters"] != iters[:n])),
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main_condense(a, arg, B, config, rank, world, local):
    """Full-condensing path: condense_batch -> dense IPM (N = 0 form) -> expand_batch.

    value: QPs/s through the three device stages, inputs resident; roofline of
    the dominant kernel (the dense IPM solve): the reference's own counted
    flops of the dense solve (identical to ours, tests/test_gpu_fcond.py) over
    its event-timed duration; e2e: the same from pinned host buffers, the
    expanded (y, pi, lam, t) and status / iterations read back.
    """
    import torch

    from paper_2003_02547_b200.condensing import (condense_batch, expand_batch,
                                                  partial_condense_batch, partial_expand_batch)
    from paper_2003_02547_b200.generators import make_batch
    from paper_2003_02547_b200.solver import get_plan, solve_ocp_qp_batch

    full = a.path == "condense"
    N1 = None if full else int(a.path.split(":", 1)[1])

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    batch = make_batch(a.cfg, batch=B)
    dev = batch.to(device)
    stream = torch.cuda.current_stream(device)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    config = dict(config, workload=config["workload"] + (
        "; full condensing + dense-QP solve + expand_solution" if full else
        f"; partial condensing N1={N1} + solve + partial_expand"))

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
    t_end = time.perf_counter() + 0.5
    while w < a.warmup or time.perf_counter() < t_end:
        step(dev)
        w += 1
    torch.cuda.synchronize()
    peak_dfma, peak_dmma = fp64_peak()
    E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [(E(), E(), (E(), E())) for _ in range(a.steps)]
    sampler = ClockSampler(index=local)
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.05)
    for e0, e1, ek in evs:
        flush.zero_()
        e0.record(stream)
        cb, rep, _ = step(dev, ek)
        e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    times = np.array([e0.elapsed_time(e1) for e0, e1, _ in evs])
    ktimes = np.array([ek[0].elapsed_time(ek[1]) for _, _, ek in evs])
    t_step = float(times.mean())
    t_k = float(ktimes.mean())
    flops = float(rep.flops.sum().item())
    iters = rep.iterations.cpu().numpy()
    status = rep.status_code.cpu().numpy()
    achieved = flops / (t_k * 1e-3) / 1e12
    plan_info = get_plan(cb).info()
    line = {"metric": METRIC, "value": world * B / (t_step * 1e-3), "unit": "solves/s",
            "n_gpus": world, "steps": a.steps, "warmup": w, "ms_per_step": t_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, BASELINE configs)", "config": config,
            "path": a.path,
            "roofline": {"bound": "tensor", "pipe": "fp64 (DFMA / DMMA)", "achieved": achieved,
                         "peak": peak_dfma, "unit": "TFLOP/s",
                         "frac": achieved / peak_dfma if peak_dfma else None, "traffic": None,
                         "kernel": ("k_ipm_solve (dense N = 0 form)" if full else
                                    f"{plan_info.get('kernel')} kernel on the condensed QPs"),
                         "work": f"reference-counted flops of the condensed solves = {flops:.4g} "
                                 f"per step over the solve kernel's {t_k:.3f} ms",
                         "kernel_share_of_step": t_k / t_step},
            "clocks": clocks, "gpu_launches": a.steps * 3, "plan": plan_info,
            "stage_ms": {"dense_solve": t_k, "condense_plus_expand": t_step - t_k},
            "condensed_dims": {"N": int(cb.dim.N), "nu": [int(v) for v in cb.dim.nu[:2]],
                               "nb": [int(v) for v in cb.dim.nb[:2]],
                               "ng": [int(v) for v in cb.dim.ng[:2]]},
            "iterations": {"min": int(iters.min()), "mean": float(iters.mean()),
                           "max": int(iters.max())},
            "status_counts": {str(int(k)): int(v) for k, v in zip(*np.unique(status, return_counts=True))}}
    if not a.no_e2e:
        hb = batch.pin_memory()
        et = []
        for i in range(max(5, a.steps // 4) + 2):
            flush.zero_()
            e0, e1 = E(), E()
            e0.record(stream)
            _, r2, (y, pi, lam, t) = step(hb)
            outs = [x.to("cpu", non_blocking=True) for x in (y, pi, lam, t, r2.status_code,
                                                            r2.iterations)]
            e1.record(stream)
            torch.cuda.synchronize()
            if i >= 2:
                et.append(e0.elapsed_time(e1))
        te = float(np.mean(et))
        line["e2e"] = {"value": world * B / (te * 1e-3), "unit": "solves/s",
                       "h2d_bytes_per_step": sum(int(v.numel()) * 8 for v in hb.fields.values()),
                       "d2h_bytes_per_step": sum(int(x.numel()) * x.element_size() for x in outs),
                       "ms_per_step": te, "steps": len(et)}
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        sys.path.insert(0, str(ROOT / "oracle"))
        import condense_oracle as co  # test infrastructure; the cpu_baseline leg only
        import oracle as orc

        from paper_2003_02547_b200 import OcpQpBatch, dense_to_ocp
        from paper_2003_02547_b200.dense import DenseQp

        orc.build()
        n = min(B, 64) if full else max(2, min(B, 8))
        qps = [batch.qp(i) for i in range(n)]
        t0 = time.perf_counter()
        dqs, maps = [], []
        if not full:
            from paper_2003_02547_b200.layout import OcpLayout

            for q in qps:
                _, blocks = co.partial_condense(q, N1)
                maps.append(blocks)
            hb = cb.numpy().select(range(n))   # condensed values (equal to the port's to 1e-12)
            ref = orc.solve(hb, arg, nthreads=os.cpu_count() or 1, trace=False)
            lay2 = OcpLayout(cb.dim)
            for i, q in enumerate(qps):
                co.partial_expand(q, maps[i], dict(layout=lay2, y=ref["y"][i], pi=ref["pi"][i],
                                                   lam=ref["lam"][i], t=ref["t"][i]))
        for q in (qps if full else []):
            dd, m = co.full_condense(q)
            dq = DenseQp(len(dd["g"]), 0, len(dd["idxb"]), len(dd["lg"]), 0)
            for f in ("H", "g", "idxb", "lb", "ub", "C", "lg", "ug", "maskl", "masku"):
                dq.set_field(f, dd[f])
            dqs.append(dense_to_ocp(dq))
            maps.append(m)
        if full:
            ref = orc.solve(OcpQpBatch.from_qps(dqs), arg, nthreads=os.cpu_count() or 1,
                            trace=False)
            for i, q in enumerate(qps):
                co.full_expand(q, maps[i], ref["y"][i], ref["lam"][i], ref["t"][i])
        tc = time.perf_counter() - t0
        line["cpu_baseline"] = {"value": n / tc, "unit": "solves/s", "cores": os.cpu_count() or 1,
                                "kind": "port",
                                "sample": f"{n} QPs of the workload: numpy "
                                          f"{'condense' if full else 'partial_condense'} + C-oracle "
                                          f"solve ({os.cpu_count()} threads) + numpy expand, "
                                          f"{tc:.2f} s"}
        line["parity_vs_oracle"] = {"qps": n,
                                    "status_mismatch": int(np.sum(ref["status"] != status[:n])),
                                    "iteration_mismatch": int(np.sum(ref["iters"] != iters[:n]))}
    if rank == 0:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
