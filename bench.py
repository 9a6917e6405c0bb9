"""Benchmark: MGRIT time-to-tolerance and fine space-time DOF/s (FP64) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl b200|reference]

A "step" is one full MGRIT solve to ||r_k|| / ||r_0|| <= 1e-10 (the
reference's SolveReport.wall_time region, mgrit.py:259-279) of the configured
BASELINE workload; value = n_x * n_t / (time per solve), whole job.  The
default workload is BASELINE configs[3] (cfg4: ERK5+U5, 8192 x 65536, m = 16,
V-cycle, GMRES-corrected SL coarse operators), the largest BASELINE config that
fits one GPU (cfg5's 137 GB iterate plus coarse levels does not).

* value / ms_per_step: iterate resident in HBM (4.3 GB for cfg4 > 126 MB L2,
  so no L2 flush is needed), CUDA events on the launching stream, max over ranks.
* e2e: the same solve through the public API ``solve(problem, config,
  initial_iterate=<pinned host tensor>)``: H2D of the iterate's live rows (the
  C-points and the rows before them -- every other row is rewritten before it
  is read; MgritSolver._upload), solve, D2H of the full final iterate, all
  inside the timed region.
* roofline: per-pass CUDA-event timing of one extra solve; algorithmic bytes and
  FP64 flops per launch of every fine-level pass over its mean launch time; the
  line's ``roofline`` is the fine pass with the largest share of the step.
* cpu_baseline: the numpy oracle (restatement of the reference, oracle/) on this
  host's cores with the reference's thread pool at 1 and cpu_count threads:
  one FCF iteration over the first n_t/16 steps, extrapolated.
* --impl reference: the same oracle as the reference arm (the reference is pure
  Python/numpy; /root/reference is absent on the GPU box), each step one such
  bounded sample on every host core.
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


def resolve_config(name: str):
    """``cfgN`` or a reduced grid of one, ``cfgN@<n_x>x<n_t>`` (tooling: per-pass
    timings of cfg5's 16384-point rows on one GPU)."""
    from paper_2209_06916_b200.configs import CONFIGS
    if "@" in name:
        base, size = name.split("@")
        n_x, n_t = (int(v) for v in size.split("x"))
        return CONFIGS[base].scaled(n_x, n_t)
    return CONFIGS[name]


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


def pass_work(cf, level, n_int, m, prog, kind, steps=None):
    """(algorithmic FP64 flops, algorithmic HBM bytes) of one launch of a fine
    explicit-stencil pass over ``n_int`` intervals:
      FC: m steps per interval (m-1 F + the C step): reads the C-point row,
          writes the C-relaxed row;
      FR: m steps: reads the C-point row and the reference C-point row, writes
          the residual row;
      CF: m steps (m-1 F + the residual tail): reads the C-point and correction
          rows once, writes every F/C row once (fine level: the iterate; the
          C-relaxed row it also stores for the next cycle is not counted).
    flops = 2 * taps per point-step (one multiply + one add per tap)."""
    n, taps = cf.n_x, len(prog.offsets)
    if prog.kind == "rk":
        # staged RK (stepping.py:355-380) per point-step: per stage one -cL stencil
        # (2 * taps) and, for SDIRK, one stage solve with the factorised operator
        # (4 flops per root of its symbol: recurrence + carry response, + 1 gain);
        # plus 2 flops per non-zero tableau entry (the Butcher sums)
        A, b = np.asarray(prog.rk_a), np.asarray(prog.rk_b)
        ns = len(b)
        solve = (4.0 * (len(prog.offsets2) - 1) + 1.0) if prog.implicit else 0.0
        butcher = 2.0 * (np.count_nonzero(np.tril(A.reshape(ns, ns), -1)) + np.count_nonzero(b))
        per_pt = ns * (2.0 * taps + solve) + butcher
    elif prog.kind == "stencil":
        per_pt = 2.0 * taps
    else:
        return None, None
    flops = per_pt * n * n_int * (m if steps is None else steps)
    rows = {"FC": 2 * n_int, "FR": 3 * n_int, "CF": n_int * m + 1 + 2 * (n_int + 1)}[kind]
    return flops, 8.0 * n * rows


def traffic_of(cf_name, pass_name):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            tr = json.load(f).get(cf_name, {}).get(pass_name)
        if tr:
            return tr["dram_read_bytes"] + tr["dram_write_bytes"], tr.get("source")
    except Exception:
        pass
    return None, None


def rooflines(cf, prob, passes, total_ms, n_int0, fp64_peak):
    """Roofline of every fine-level pass from its CUDA-event launch times: the
    bound is whichever of HBM bytes / peak and FP64 flops / issue bound is
    larger.  Exact mode issues DMUL + DADD per tap, so its FP64 issue bound is
    half the DFMA peak (reported as ``frac_of_issue_bound``)."""
    from paper_2209_06916_b200 import mgrit as _mg
    elided = bool(_mg.ELIDE_OPENING_F_RELAX)
    hbm_peak, peak_kind = peaks()
    prog = prob.steppers[0].program
    out = {}
    for kind in ("FC", "FR", "CF"):
        name = f"L0.{kind}"
        if name not in passes:
            continue
        cnt, ms = passes[name]
        # the opening FC pass of iterations >= 2 is one C-step per interval from the stored
        # last F-point (mgrit.ELIDE_OPENING_F_RELAX): average steps per launch of the solve
        m0 = prob.m[0]
        steps = (m0 + (cnt - 1)) / cnt if (kind == "FC" and elided and cnt > 1) else None
        flops, nbytes = pass_work(cf, 0, n_int0, m0, prog, kind, steps)
        if flops is None:
            continue
        t = ms / cnt / 1e3
        # exact explicit stencils issue DMUL + DADD per tap; staged RK mixes fused solves
        # with exact stencil / tableau sums and is reported against the DFMA peak
        issue = fp64_peak * (0.5 if (prog.exact and prog.kind == "stencil") else 1.0)
        fp64_bound = flops / (issue * 1e9) >= nbytes / (hbm_peak * 1e9)
        traffic, tsrc = traffic_of(cf.name, name)
        if fp64_bound:
            ach = flops / t / 1e12
            r = {"bound": "fp64", "achieved": round(ach, 3), "peak": round(fp64_peak / 1e3, 3),
                 "unit": "TFLOP/s", "frac": round(ach * 1e3 / fp64_peak, 4),
                 "frac_of_issue_bound": round(ach * 1e3 / issue, 4),
                 "peak_source": "measured live: DFMA probe (mgb_fp64_peak), 2 flop per DFMA",
                 "algorithmic_flops": flops}
        else:
            ach = nbytes / t / 1e9
            r = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                 "frac": round(ach / hbm_peak, 4), "peak_source": peak_kind + " (MEASURED_PEAKS.json)"}
        if steps is not None:
            r["steps_per_launch_avg"] = round(steps, 3)
        r.update({"kernel": f"relax kernel {name}", "algorithmic_bytes": nbytes,
                  "launch_ms": round(t * 1e3, 4), "traffic": traffic, "traffic_source": tsrc,
                  "share_of_step": round(ms / total_ms, 4)})
        out[name] = r
    return out


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


def bench_config(cf) -> dict:
    """The ``config`` object of every bench line: identical in both arms and at
    every N (per-run solve details go under ``solve``)."""
    it_bytes = 8 * (cf.n_t + 1) * cf.n_x
    return {"workload": workload(cf), "n_x": cf.n_x, "n_t": cf.n_t, "m": cf.m,
            "cycle": cf.cycle, "tol": 1e-10, "max_iters": 30,
            "l2": (f"iterate {it_bytes / 1e6:.0f} MB > 126 MB L2: inputs larger than L2, "
                   "no flush needed") if it_bytes > 126e6 else "iterate fits L2",
            "arith": "exact (mul-then-add, reference tap order)"}


def one_level_profile(solver, one_solve):
    solver.profile = []
    one_solve()
    passes = solver.profile_summary()
    solver.profile = None
    return passes


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
    cf = resolve_config(args.config)
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
    dof = cf.n_x * cf.n_t
    value = dof / (ms_step / 1e3)

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
    ubytes = u_host.nbytes
    del host

    # per-pass breakdown (CUDA events around every launch of one extra solve)
    passes = one_level_profile(solver, one_solve)
    total_ms = sum(ms for _, ms in passes.values())
    fp64_peak = fp64_peak_gflops()
    roofs = rooflines(cf, prob, passes, total_ms, solver.levels[0].n_int, fp64_peak)
    # the roofline line: the fine-level pass with the largest share of the step
    top = max(roofs.items(), key=lambda kv: kv[1]["share_of_step"]) if roofs else None
    breakdown = {k: {"launches": c, "ms": round(ms, 4), "share": round(ms / total_ms, 4)}
                 for k, (c, ms) in sorted(passes.items(), key=lambda kv: -kv[1][1])}
    dom = max(passes.items(), key=lambda kv: kv[1][1])
    levels = {}
    for k, (c, ms) in passes.items():
        lv = k.split(".")[0]
        levels[lv] = round(levels.get(lv, 0.0) + ms / total_ms, 4)

    result = {
        "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": value, "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cf),
        "solve": {"iterations": rep.iterations, "converged": rep.converged,
                  "final_ratio": rep.residual_norms[-1] / rep.residual_norms[0],
                  "time_to_tolerance_s": ms_step / 1e3, "parallelism": "single GPU"},
        "e2e": {"value": dof / e2e_s, "unit": "DOF/s",
                "h2d_bytes_per_step": int(esol.last_upload_bytes),
                "d2h_bytes_per_step": ubytes + 8 * len(rep_e2e.residual_norms),
                "seconds": e2e_s,
                "note": "P.solve(problem, config, initial_iterate=<pinned host tensor>): H2D of "
                        "the rows the solve reads before rewriting them (C-points and the rows "
                        "before them; MgritSolver._upload), solve, D2H of the full final "
                        "iterate (in-place semantics), all inside the timed region"},
        "gpu_launches": launches,
        "roofline": dict(top[1], pass_name=top[0]) if top else None,
        "roofline_passes": roofs,
        "dominant_pass": {"name": dom[0], "share": round(dom[1][1] / total_ms, 4)},
        "level_shares": levels,
        "passes": breakdown,
        "clocks": clk.summary(),
    }
    if not args.no_fast:
        result["fast_mode"] = fast_mode_line(args, cf, cfg, u_pristine, u, rep, fp64_peak)
    if rank == 0 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(cf)
    print(json.dumps(result), flush=True)


def fast_mode_line(args, cf, cfg, u_pristine, u, rep_exact, fp64_peak):
    """Secondary measurement: the same solve with the explicit stencils in DFMA
    ("fast") arithmetic (``stepping.EXACT_ARITHMETIC = False``: one fused
    multiply-add per tap instead of the reference's rounded product + rounded
    sum).  Results differ from exact mode by rounding only; the line reports the
    deviation of the residual history next to the timing and the fine-pass
    rooflines against the full DFMA peak."""
    import torch
    import paper_2209_06916_b200 as P
    from paper_2209_06916_b200 import stepping
    stepping.EXACT_ARITHMETIC = False
    try:
        prob = cf.problem()
        solver = P.MgritSolver(prob, cfg)

        def one_solve():
            u.copy_(u_pristine)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            rep = solver.solve(u)
            e.record()
            torch.cuda.synchronize()
            return rep, s.elapsed_time(e)

        for _ in range(min(args.warmup, 3)):
            one_solve()
        times = []
        for _ in range(max(3, min(args.steps, 5))):
            rep, ms = one_solve()
            times.append(ms)
        passes = one_level_profile(solver, one_solve)
        total_ms = sum(ms for _, ms in passes.values())
        roofs = rooflines(cf, prob, passes, total_ms, solver.levels[0].n_int, fp64_peak)
    finally:
        stepping.EXACT_ARITHMETIC = True
    r0 = rep_exact.residual_norms[0]
    dev = max(abs(a - b) / r0 for a, b in zip(rep.residual_norms, rep_exact.residual_norms))
    ms_step = float(np.mean(times))
    return {"arith": "DFMA (one fused multiply-add per tap)", "ms_per_step": ms_step,
            "value": cf.n_x * cf.n_t / (ms_step / 1e3), "iterations": rep.iterations,
            "converged": rep.converged,
            "history_dev_vs_exact_over_r0": dev if rep.iterations == rep_exact.iterations else None,
            "roofline_passes": {k: {kk: v[kk] for kk in ("bound", "achieved", "peak", "unit", "frac",
                                                         "launch_ms", "share_of_step")}
                                for k, v in roofs.items()}}


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
    sol.solve(ud)
    host.copy_(ud)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], device="cuda", dtype=torch.float64)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    nbytes = torch.tensor([float(u_host.nbytes)], device="cuda", dtype=torch.float64)
    dist.all_reduce(nbytes)
    lt = torch.tensor([float(launches)], device="cuda", dtype=torch.float64)
    dist.all_reduce(lt)
    # per-pass breakdown of this rank's block (CUDA events around every launch)
    eng.profile = []
    one_solve()
    passes = eng.profile_summary()
    eng.profile = None
    total_ms = sum(ms for _, ms in passes.values()) or 1.0
    roofs = rooflines(cf, prob, passes, total_ms, sol.nb, fp64_peak_gflops())
    top = max(roofs.items(), key=lambda kv: kv[1]["share_of_step"]) if roofs else None
    dof = cf.n_x * cf.n_t
    result = {
        "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": dof / (ms_step / 1e3), "unit": "DOF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cf),
        "solve": {"iterations": rep.iterations, "converged": rep.converged,
                  "final_ratio": rep.residual_norms[-1] / rep.residual_norms[0],
                  "time_to_tolerance_s": ms_step / 1e3,
                  "parallelism": f"time-sharded x{world} (levels 0..{sol.ls - 1} in interval "
                                 f"blocks per rank, levels >= {sol.ls} on rank 0)"},
        "e2e": {"value": dof / float(te.item()), "unit": "DOF/s",
                "h2d_bytes_per_step": int(nbytes.item()),
                "d2h_bytes_per_step": int(nbytes.item())},
        "gpu_launches": int(lt.item()),
        "roofline": dict(top[1], pass_name=top[0], rank=0) if top else None,
        "roofline_passes": roofs,
        "passes": {k: {"launches": c, "ms": round(ms, 4), "share": round(ms / total_ms, 4)}
                   for k, (c, ms) in sorted(passes.items(), key=lambda kv: -kv[1][1])},
        "clocks": clk.summary(),
        "cpu_baseline_note": "the CPU baseline runs on rank 0 at N = 1 only",
    }
    dist.barrier()
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(result), flush=True)


# ------------------------------------------------------------ CPU baseline

def sample_nt(cf) -> int:
    """n_t of the bounded CPU sample: the first n_t / 16 steps of the workload
    (same n_x, scheme, m and coarse operators; one level fewer -- cfg4: 4 of its
    5 levels), so a sample iteration takes seconds instead of minutes."""
    return max(cf.n_t // 16, cf.m * cf.m)


def oracle_sample(cf, threads=1, n_t=None):
    """One FCF V-cycle iteration (+ initial and final norm) of the workload's
    bounded sample on the oracle with the reference's row-chunk thread pool
    (mgrit.py:113-129).  Returns (seconds, n_t of the sample)."""
    from oracle import mgrit_oracle as O
    from paper_2209_06916_b200.configs import seeded_u0
    n_t = n_t or sample_nt(cf)
    O.ROLL_LIMIT = 64 if cf.p == 5 else 16
    steps, fac, _ = O.build_hierarchy(cf.family, cf.p, cf.c, cf.n_x, n_t, cf.m, cf.cycle,
                                      cf.coarse, fine_mode="staged" if cf.family == "sdirk"
                                      else "assembled")
    mg = O.Mgrit(steps, fac, n_t, seeded_u0(cf.u0, cf.n_x), cycle=cf.cycle, threads=threads)
    u = mg.initial_state()
    t0 = time.perf_counter()
    mg.solve(u, max_iters=1)
    return time.perf_counter() - t0, n_t


def extrapolate(cf, sample_s, n_t_sample):
    """Time to tolerance of the full workload from one sample iteration:
    x (n_t / n_t_sample) for the time axis, x the reference's iteration count."""
    return sample_s * (cf.n_t / n_t_sample) * reference_iterations(cf)


def cpu_baseline(cf):
    rows = []
    for thr in sorted({1, os.cpu_count() or 1}):
        wall, nts = oracle_sample(cf, threads=thr)
        tts = extrapolate(cf, wall, nts)
        rows.append({"threads": thr, "sample_s": round(wall, 3),
                     "time_to_tolerance_s_extrapolated": round(tts, 1),
                     "value": cf.n_x * cf.n_t / tts})
    best = max(rows, key=lambda r: r["value"])
    return {"value": best["value"], "unit": "DOF/s", "cores": best["threads"], "kind": "port",
            "sample": (f"numpy oracle (restatement of the reference, pinned bitwise to it): one "
                       f"FCF V-cycle iteration + norms of {cf.name} over its first "
                       f"{sample_nt(cf)} of {cf.n_t} time steps, extrapolated x "
                       f"{cf.n_t // sample_nt(cf)} (time axis) x {reference_iterations(cf)} "
                       f"iterations (the reference's count); threads = the reference's "
                       f"row-chunk pool (mgrit.py:113-129)"),
            "extrapolated": True, "rows": rows, "cpu_count": os.cpu_count()}


def run_reference(args):
    """The reference arm: the reference's CPU path (the pinned numpy oracle;
    the reference is pure Python and absent on the GPU box) on this host's
    cores.  Each step is one bounded sample of the workload (one FCF iteration
    over the first n_t / 16 time steps, the reference's thread pool with every
    host core); value = the extrapolated time-to-tolerance DOF/s."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    from paper_2209_06916_b200.configs import CONFIGS
    cf = resolve_config(args.config)
    thr = os.cpu_count() or 1
    for _ in range(args.warmup):
        oracle_sample(cf, threads=thr)
    times = []
    for _ in range(max(1, args.steps)):
        wall, nts = oracle_sample(cf, threads=thr)
        times.append(wall)
    per_sample = float(np.mean(times))
    tts = extrapolate(cf, per_sample, nts)
    value = cf.n_x * cf.n_t / tts
    sample = (f"numpy oracle (the reference's algorithm, pinned bitwise): each step = one FCF "
              f"V-cycle iteration + norms of {cf.name} over its first {nts} of {cf.n_t} time "
              f"steps with the reference's row-chunk thread pool at {thr} threads; value "
              f"extrapolated x {cf.n_t // nts} (time axis) x {reference_iterations(cf)} "
              f"iterations")
    print(json.dumps({
        "impl": "reference", "metric": "MGRIT time-to-tolerance fine space-time DOF/s (FP64)",
        "value": value, "unit": "DOF/s", "n_gpus": int(os.environ.get("WORLD_SIZE", 1)),
        "steps": len(times), "warmup": args.warmup, "ms_per_step": per_sample * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(cf),
        "extrapolated": {"time_to_tolerance_s": tts, "factor_time_axis": cf.n_t // nts,
                         "iterations": reference_iterations(cf),
                         "note": "ms_per_step is the measured sample; value is extrapolated"},
        "cpu_baseline": {"value": value, "unit": "DOF/s", "cores": thr, "kind": "port",
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
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fast", action="store_true", help="skip the secondary DFMA-mode solve")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
