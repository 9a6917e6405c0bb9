"""Benchmark: MGRIT time-to-tolerance and fine space-time DOF/s (FP64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl b200|reference]

A "step" is one full MGRIT solve to ||r_k|| / ||r_0|| <= 1e-10 (the
reference's SolveReport.wall_time region, mgrit.py:259-279) of the configured
BASELINE workload; value = n_x * n_t / (time per solve), whole job.

* value / ms_per_step: iterate resident in HBM (537 MB for cfg2 > 126 MB L2,
  so no L2 flush is needed), CUDA events on the launching stream, max over ranks.
* e2e: the same solve through the public API ``mgrit.solve(problem, config,
  initial_iterate=<pinned host tensor>)``: H2D of the iterate's live rows (the
  C-points and the rows before them -- every other row is rewritten before it
  is read; MgritSolver._upload), solve, D2H of the full final iterate, all
  inside the timed region.
* roofline: per-pass CUDA-event timing of one extra solve; the dominant pass's
  algorithmic bytes (or FP64 flops) per launch over its mean launch time.
* cpu_baseline: the numpy oracle (restatement of the reference, oracle/) on this
  host's cores: one full V-cycle iteration of the same workload, extrapolated
  with the iteration count to a time-to-tolerance.
* --impl reference: the same oracle as the reference arm (the reference is
  pure Python/numpy; /root/reference is absent on the GPU box).
Multi-GPU (torchrun, N > 1): ONE time-sharded solve of the workload over the N
ranks (strong scaling): every level whose intervals split over the ranks is
sharded in contiguous interval blocks, one boundary C-point row per FC pass and
level goes to the right neighbour over NCCL, the first level with too few
intervals is gathered to rank 0 with the rest of the cycle
(paper_2209_06916_b200/distributed.py).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

HBM_FALLBACK_GBS = 6650.0


def workload(cf) -> str:
    """The workload named in every bench line (both arms, every N)."""
    return (f"{cf.name}: {cf.family.upper()}{cf.p}+U{cf.p} c={cf.c} n_x={cf.n_x} n_t={cf.n_t} "
            f"m={cf.m} {cf.cycle} {cf.coarse} coarse op, FCF, tol 1e-10, u0={cf.u0}")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    in-process every 5 ms (nvidia-smi as a fallback), median SM clock of the
    samples and the union of the slowdown reasons seen."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index: int, period: float = 0.005):
        self.index = index
        self.period = period
        self.samples = []  # (sm_mhz, max_mhz, reasons bitmask)
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._max = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = float(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
            try:
                rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self._h))
            except Exception:
                rs = int(nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h))
            return sm, self._max, rs
        out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                              "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        return float(f[0]), float(f[1]), int(f[2], 16)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = set()
        for _, _, rs in self.samples:
            for name, attr in self.REASONS:
                bit = getattr(self._nvml, attr, None) if self._nvml else None
                if bit is None:
                    bit = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                           "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4,
                           "hw_power_brake": 0x80}[name]
                if rs & bit:
                    reasons.add(name)
        return {"sm_mhz": float(np.median([s[0] for s in self.samples])),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": sorted(reasons),
                "samples": len(self.samples),
                "source": "nvml 5 ms" if self._nvml is not None else "nvidia-smi"}


def algorithmic_work(cf, solver, name):
    """(bound, algorithmic bytes or FP64 flops per launch) of one relax pass."""
    lev = int(name[1]) if name[0] == "L" and name[1].isdigit() else 0
    n = cf.n_x
    if lev >= len(solver.levels):
        return "latency", None
    L = solver.levels[lev]
    nI, m = L.n_int, L.m
    prog = solver.problem.steppers[lev].program
    kind = name.split(".")[1]
    if prog.kind == "stencil":
        taps = len(prog.offsets)
        flops = 2.0 * taps * n * nI * (m if kind != "R" else 1)
        if kind == "CF":  # all F/C rows written once + C-point and correction rows read once
            return "hbm", 8.0 * n * (nI * m + 1 + 2 * (nI + 1))
        if kind in ("FC", "FR"):
            return "fp64", flops
        return "hbm", 8.0 * n * 2 * nI
    return "latency", None


def fp64_peak_gflops() -> float:
    """Measured FP64 DFMA throughput of this GPU (GFLOP/s), CUDA events."""
    import ctypes
    import torch
    from paper_2209_06916_b200 import _native
    lib = _native.load()
    fl = ctypes.c_double()
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    lib.mgb_fp64_peak(1000, ctypes.byref(fl), stream)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        lib.mgb_fp64_peak(20000, ctypes.byref(fl), stream)
        e.record()
        torch.cuda.synchronize()
        best = max(best, fl.value / (s.elapsed_time(e) / 1e3) / 1e9)
    return best


def run_gpu(args):
    import torch
    import torch.distributed as dist
    import paper_2209_06916_b200 as P
    from paper_2209_06916_b200 import _native
    from paper_2209_06916_b200.configs import CONFIGS

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cf = CONFIGS[args.config]
    prob = cf.problem()
    cfg = P.MgritConfig(nu=1, cycle=cf.cycle, tol=1e-10, max_iters=30, rng_seed=0)
    if world > 1:
        return run_sharded(args, cf, prob, cfg, rank, world, local)
    solver = P.MgritSolver(prob, cfg)
    u_host = solver.initial_state()
    u_pristine = torch.from_numpy(u_host).to("cuda")
    u = torch.empty_like(u_pristine)
    stream = torch.cuda.current_stream()

    def one_solve():
        u.copy_(u_pristine)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        rep = solver.solve(u)
        e.record(stream)
        torch.cuda.synchronize()
        return rep, s.elapsed_time(e)

    for _ in range(args.warmup):
        rep, _ = one_solve()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _native.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            rep, ms = one_solve()
            times.append(ms)
    torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms_step = float(np.mean(times))
    if world > 1:
        t = torch.tensor([ms_step], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    dof = cf.n_x * cf.n_t
    value = world * dof / (ms_step / 1e3)

    # e2e through the public API with a pinned host iterate
    host = torch.from_numpy(u_host).pin_memory()
    e2e_times = []
    for _ in range(max(3, min(args.steps, 5))):
        host.copy_(torch.from_numpy(u_host))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        esol = P.MgritSolver(prob, cfg)
        rep_e2e = esol.solve(host)  # == P.solve(prob, cfg, initial_iterate=host)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    e2e_s = float(np.median(e2e_times))  # host-side PCIe timing varies run to run
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    ubytes = u_host.nbytes

    # per-pass breakdown -> roofline of the dominant pass
    solver.profile = []
    rep_p, _ = one_solve()
    passes = solver.profile_summary()
    solver.profile = None
    total_ms = sum(ms for _, ms in passes.values())
    hbm_peak, peak_kind = peaks()
    dom = max(passes.items(), key=lambda kv: kv[1][1])
    roof = None
    fine_cf = passes.get("L0.CF")
    bound, work = algorithmic_work(cf, solver, "L0.CF") if fine_cf else (None, None)
    if fine_cf and work:
        per_launch_s = fine_cf[1] / fine_cf[0] / 1e3
        ach = work / per_launch_s / 1e9
        traffic = None
        try:
            with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
                tr = json.load(f).get("L0.CF")
            if tr:
                traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
        except Exception:
            pass
        roof = {"bound": "hbm", "kernel": "relax_kernel L0.CF (correct + F-relax + residual)",
                "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "peak_source": peak_kind,
                "algorithmic_bytes": work, "traffic": traffic,
                "traffic_source": "profiles/traffic.json (ncu --set full, one launch)",
                "share_of_step": round(fine_cf[1] / total_ms, 4)}
    roof_fp64 = None
    fine_fc = passes.get("L0.FC")
    _, flops = algorithmic_work(cf, solver, "L0.FC") if fine_fc else (None, None)
    if fine_fc and flops:
        fp64_peak = fp64_peak_gflops()
        ach = flops / (fine_fc[1] / fine_fc[0] / 1e3) / 1e9
        roof_fp64 = {"bound": "fp64", "kernel": "relax_kernel L0.FC (F-relax + C-relax, exact mode)",
                     "achieved": round(ach, 1), "peak": round(fp64_peak, 1), "unit": "GFLOP/s",
                     "frac": round(ach / fp64_peak, 4),
                     "peak_source": "measured live: DFMA probe (mgb_fp64_peak), 2 flop/DFMA",
                     "note": "exact mode issues DMUL+DADD per tap (2 flop in 2 issue slots): "
                             "the pipe-time bound is half the DFMA peak"}
    breakdown = {k: {"launches": c, "ms": round(ms, 4), "share": round(ms / total_ms, 4)}
                 for k, (c, ms) in sorted(passes.items(), key=lambda kv: -kv[1][1])}

    result = {
        "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(cf),
                   "iterations": rep.iterations, "converged": rep.converged,
                   "final_ratio": rep.residual_norms[-1] / rep.residual_norms[0],
                   "time_to_tolerance_s": ms_step / 1e3,
                   "parallelism": "replicas" if world > 1 else "single",
                   "l2": "iterate 537MB > L2; no flush needed" if ubytes > 126e6 else "iterate fits L2",
                   "arith": "exact (mul-then-add, reference tap order)"},
        "e2e": {"value": world * dof / e2e_s, "unit": "DOF/s",
                "h2d_bytes_per_step": int(esol.last_upload_bytes),
                "d2h_bytes_per_step": ubytes + 8 * len(rep_e2e.residual_norms),
                "seconds": e2e_s,
                "note": "H2D moves the rows the solve reads before rewriting them (C-points "
                        "and the rows before them; MgritSolver._upload), D2H the full final "
                        "iterate (in-place semantics)"},
        "gpu_launches": launches,
        "roofline": roof,
        "roofline_fp64": roof_fp64,
        "dominant_pass": {"name": dom[0], "share": round(dom[1][1] / total_ms, 4)},
        "passes": breakdown,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cf, rep.iterations)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def run_sharded(args, cf, prob, cfg, rank, world, local):
    """N > 1: one time-sharded solve of the workload over all ranks (strong
    scaling): interval blocks per rank on every sharded level, boundary-row
    exchange over NCCL, the remaining coarse levels on rank 0
    (paper_2209_06916_b200/distributed.py)."""
    import torch
    import torch.distributed as dist
    from paper_2209_06916_b200 import _native
    from paper_2209_06916_b200.distributed import GpuEngine, ShardedMgritSolver, initial_rows

    eng = GpuEngine(prob, cfg)
    sol = ShardedMgritSolver(prob, cfg, eng)
    r0, r1 = sol.local_rows()
    u_host = initial_rows(cfg.rng_seed, r0, r1, cf.n_x, prob.u0)
    pristine = torch.from_numpy(u_host).to("cuda")
    u = torch.empty_like(pristine)

    def one_solve():
        u.copy_(pristine)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        rep = sol.solve(u)
        e.record()
        torch.cuda.synchronize()
        return rep, s.elapsed_time(e)

    for _ in range(args.warmup):
        one_solve()
    launches0 = _native.launch_count()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            rep, ms = one_solve()
            times.append(ms)
    launches = _native.launch_count() - launches0
    t = torch.tensor([float(np.mean(times))], device="cuda", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item())
    # e2e: pinned host block -> device -> sharded solve -> host, per rank
    host = torch.from_numpy(u_host).pin_memory()
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    ud = host.to("cuda", non_blocking=True)
    rep_e = sol.solve(ud)
    host.copy_(ud)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    nbytes = torch.tensor([float(u_host.nbytes)], device="cuda", dtype=torch.float64)
    dist.all_reduce(nbytes)
    lt = torch.tensor([float(launches)], device="cuda", dtype=torch.float64)
    dist.all_reduce(lt)
    dof = cf.n_x * cf.n_t
    result = {
        "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": dof / (ms_step / 1e3), "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload(cf),
                   "iterations": rep.iterations, "converged": rep.converged,
                   "parallelism": f"time-sharded x{world} (levels 0..{sol.ls - 1} in interval "
                                  f"blocks per rank, levels >= {sol.ls} on rank 0)"},
        "e2e": {"value": dof / float(te.item()), "unit": "DOF/s",
                "h2d_bytes_per_step": int(nbytes.item()),
                "d2h_bytes_per_step": int(nbytes.item())},
        "gpu_launches": int(lt.item()),
        "roofline": None,
        "clocks": clk.summary(),
    }
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


def oracle_sample(cf, n_iters_sample=1):
    """One V-cycle iteration (+ initial norm) of the workload on the oracle."""
    from oracle import mgrit_oracle as O
    O.ROLL_LIMIT = 64 if cf.p == 5 else 16
    steps, fac, _ = O.build_hierarchy(cf.family, cf.p, cf.c, cf.n_x, cf.n_t, cf.m, cf.cycle,
                                      cf.coarse, fine_mode="staged" if cf.family == "sdirk"
                                      else "assembled")
    from paper_2209_06916_b200.configs import seeded_u0
    u0 = seeded_u0(cf.u0, cf.n_x)
    mg = O.Mgrit(steps, fac, cf.n_t, u0, cycle=cf.cycle)
    u = mg.initial_state()
    t0 = time.perf_counter()
    out = mg.solve(u, max_iters=n_iters_sample)
    return time.perf_counter() - t0, out


def cpu_baseline(cf, iterations):
    wall, out = oracle_sample(cf)
    per_solve = wall * max(iterations, 1)  # initial norm ~1/3 iteration: conservative
    return {"value": cf.n_x * cf.n_t / per_solve, "unit": "DOF/s", "cores": 1, "kind": "port",
            "sample": f"oracle (numpy restatement of the reference) on this host: 1 FCF "
                      f"V-cycle iteration + initial norm of {cf.name} at full size took "
                      f"{wall:.2f}s, x {iterations} iterations to tolerance",
            "threads": 1, "cpu_count": os.cpu_count()}


def run_reference(args):
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from paper_2209_06916_b200.configs import CONFIGS
    cf = CONFIGS[args.config]
    iters = reference_iterations(cf)
    budget = 180.0
    times = []
    for i in range(max(1, args.steps)):
        wall, _ = oracle_sample(cf)
        times.append(wall)
        if sum(times) > budget:
            break
    per_iter = float(np.mean(times))
    per_solve = per_iter * iters
    value = cf.n_x * cf.n_t / per_solve
    sample = (f"numpy oracle: each step = 1 FCF iteration (+ initial norm) of {cf.name} at full "
              f"size; {len(times)} of {args.steps} steps run (180 s budget); extrapolated "
              f"x {iters} iterations (the reference's own count); threads=1, the reference's "
              f"fastest setting (its row-chunk thread pool is GIL-bound and slower, SURVEY 6.2)")
    print(json.dumps({
        "impl": "reference", "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": value, "unit": "DOF/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)),
        "steps": len(times), "warmup": 0, "ms_per_step": per_solve * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload(cf)},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": 1, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": "DOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def reference_iterations(cf):
    """Iteration count of the reference on this workload (golden fixture made by
    running the real reference; see tests/golden/make_golden.py)."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "histories.json")) as f:
            return int(json.load(f)[cf.name]["iterations"])
    except Exception:
        return {"cfg1": 11, "cfg2": 11, "cfg3": 22, "cfg4": 21}.get(cf.name, 11)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
