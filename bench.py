"""Benchmark of the MOT hot path (driver contract: one JSON line on rank 0).

Workload (default --config 2 = BASELINE.json configs[2], the configuration the
metric is quoted on at 1/2/4/8 B200): 5120-element jittered unit icosphere,
Burton-Miller d=1, Dirichlet, Nt=256, direct (banded) history convolution,
rows sharded over the GPUs.  A bench *step* is one complete time loop: the
Nt-1 = 255 MOT time steps of the configuration.

  value   MOT time-steps/s of the time loop, banded coefficient store resident
          in HBM (1.5 GB, i.e. larger than the 126 MB L2: no flush needed),
          device time (CUDA events on the library stream) max over ranks.
  e2e     the same metric through the public API march(spec, mats=store) with
          plain per-step data callables (the reference's contract): Greville
          sampling on the host, H2D of the known data, the loop, D2H of u, q,
          tau, sigma -- every call.  e2e_vectorised_data / e2e_device_boundary_data
          report the scenario's vectorised and device-side data sources beside it.
  e2e_with_assembly  cold march(spec): store build + assembly + loop + copies.
  roofline  K2 (history convolution): the store read once per launch (16 B x
          N_band) / average launch time measured with CUDA events around every
          K2 launch of the timed region, against the measured HBM copy
          bandwidth; `traffic` = ncu DRAM bytes of that kernel at that kb.
          `blocking` reports the kb MOT steps one store read serves.
  assembly  K1 (coefficient fill) evals/s; its roofline fraction is ncu's FP64-
          pipe utilisation at this configuration (profiles/k1_fill.json).
  cpu_baseline  the C oracle port (oracle/) of the reference's march (sigma/tau
          lag-CSR form) on the host cores: the complete loop of the full problem.
  --impl reference  the same port, a bench step = a chunk of consecutive MOT
          steps of the full-problem loop (assembly outside the timed region).
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

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "MOT time-steps/s"
# SURVEY 8(d) K1 cost model: FP64-pipe instruction-equivalents per (i,j,gamma) evaluation
K1_COST = {("uw", 1): 3957, ("bm", 1): 6513, ("uw", 2): 4713, ("bm", 2): 10071,
           ("uw", 3): 4689, ("bm", 3): 9177}
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        samples = [[v.strip() for v in l.split(",")] for l in self.lines]
        samples = [s for s in samples if len(s) >= 6]
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = sorted(v for v in (num(s[0]) for s in samples) if v is not None)
        mx = max((v for v in (num(s[1]) for s in samples) if v is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in samples for k in range(4) if s[2 + k].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def per_step_spec(spec):
    """The spec with its data callables as plain per-step functions (no vectorised
    or device forms): what a reference user passes (marching.py:33-64)."""
    import dataclasses
    import warnings

    def plain(fn):
        return None if fn is None else (lambda t, fn=fn: fn(t))
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return dataclasses.replace(spec, u_data=plain(spec.u_data), q_data=plain(spec.q_data))


def cpu_marcher(spec):
    """The oracle port (C/OpenMP) of the reference's march on the WHOLE problem:
    lag-CSR assembly of every row (marching.py:132-181), then a stateful time
    loop (marching.py:292-338) that bench.py advances in bounded chunks."""
    from oracle import oracle
    oracle.build()
    uk, qk = _greville(spec)
    thr = 1e6 * max(spec.blowup_reference, 1e-30)
    return oracle.Marcher(spec.mesh.vertices, spec.mesh.triangles, spec.phi, spec.bie, spec.basis.d,
                          spec.c, spec.basis.dt, spec.nt, uk, qk, threshold=thr)


def _greville(spec):
    from paper_2111_05205_b200 import marching
    return marching.greville_samples(spec)


def cpu_full_loop(spec):
    """cpu_baseline of our arm: the complete (nt-1)-step loop of the oracle port on
    the full problem, timed on the host cores (assembly reported, not in value)."""
    from oracle import oracle
    M = cpu_marcher(spec)
    try:
        n, t, done = M.run(spec.nt - 1)
    finally:
        t_asm = M.t_asm
        M.close()
    ns = spec.mesh.n_elements
    return {"value": n / t, "unit": "steps/s", "cores": oracle.num_threads(), "kind": "port",
            "sample": (f"the complete loop: all {n} MOT steps of the full {ns}-element problem "
                       f"(sigma/tau lag-CSR SpMVs + Gauss-Seidel solve + residual test), "
                       f"oracle port (C/OpenMP) of marching.march; loop {t:.1f} s; lag-CSR assembly "
                       f"of all rows {t_asm:.1f} s (not in value)"),
            "loop_s": t, "assembly_s": t_asm, "steps": n}


def run_reference(args, world, rank):
    """--impl reference: the reference's algorithm on the host cores (oracle port,
    C/OpenMP, all host threads).  The lag CSR of the whole problem is assembled
    once (outside the timed region); a bench step is one chunk of `--ref-chunk`
    consecutive MOT steps of the real full-problem loop, which continues across
    bench steps and restarts from step 1 when it reaches the end."""
    from oracle import oracle
    from paper_2111_05205_b200 import scenarios
    if rank != 0:
        return
    spec = scenarios.build_spec(args.config)
    nt = spec.nt
    chunk = args.ref_chunk or -(-(nt - 1) // 8)
    t0 = time.perf_counter()
    M = cpu_marcher(spec)
    t_setup = time.perf_counter() - t0

    def one_chunk():
        left, steps, secs = chunk, 0, 0.0
        while left > 0:
            n, t, done = M.run(left)
            steps, secs, left = steps + n, secs + t, left - n
            if done:
                M.reset()
        return steps, secs

    for _ in range(args.warmup):
        one_chunk()
    tot_steps, tot_s = 0, 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        n, t = one_chunk()
        tot_steps += n
        tot_s += t
    wall = time.perf_counter() - t0
    M.close()
    value = tot_steps / tot_s
    cores = oracle.num_threads()
    sample = (f"{args.steps} chunks of {chunk} consecutive MOT steps of the full "
              f"{spec.mesh.n_elements}-element loop ({nt - 1} steps, restarted at the end) after "
              f"{args.warmup} warm-up chunks; oracle port (C, OpenMP) of marching.march in the "
              f"reference's sigma/tau lag-CSR form; lag-CSR assembly of all rows {M.t_asm:.1f} s, "
              f"outside the timed region")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded scenario)",
        "config": {"workload": scenarios.DESCRIPTION[args.config], "ns": spec.mesh.n_elements,
                   "nt": nt, "mot_steps_per_bench_step": chunk, "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": "steps/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "timed_wall_s": wall, "setup_s": t_setup,
    }
    print(json.dumps(line), flush=True)


def m2l_flops(plan, nt: int, d: int) -> float:
    """Executed M2L FLOPs of the whole FMM loop: per interaction pair and level tick
    2 * 256 * (64 NT + 256 d) -- the NT = (mu+1)(pt-1)+1 distinct near-future time
    offsets (shared rows of consecutive lags) plus the d derivative operators
    (csrc/fmm.cu m2l_dmma_kernel); level leaf - j ticks when the low j bits of the
    leaf tick are all 1 (csrc/fmm.cu tick())."""
    from paper_2111_05205_b200 import fmm_plan
    sch = fmm_plan.step_schedule(plan, nt)
    n_ticks = int(sch["ticks_before"][nt - 1]) + 1
    rows = 64 * ((plan.mu + 1) * (plan.pt - 1) + 1) + 256 * d
    total = 0.0
    for L, lev in plan.levels.items():
        j = plan.leaf - L
        ticks = sum(1 for k in range(n_ticks) if (k & ((1 << j) - 1)) == (1 << j) - 1)
        total += 2.0 * 256 * rows * len(lev.il_obs) * ticks
    return total


def run_fmm(args, world, rank, local, ctx, spec, barrier, max_over_ranks):
    """Configs 3-4 on the interpolation FMM (fmm.fast_march's store, target-cell
    sharded over the ranks): loop steps/s resident, e2e through march(), and the
    M2L DGEMM FLOP rate of the whole loop against the live FP64 peak."""
    import ctypes as C
    import time as _time
    from paper_2111_05205_b200 import _lib, fmm, fmm_plan, marching, scenarios
    conf = fmm_plan.FmmConfig(ps=4, pt=4, leaf_capacity=20)
    t0 = _time.perf_counter()
    plan = fmm_plan.build_plan(spec, conf)
    t_plan = _time.perf_counter() - t0
    store = fmm.FmmStore(spec, conf, plan=plan, nranks=world, rank=rank).assemble()
    info = store.info()
    ns, nt = spec.mesh.n_elements, spec.nt
    thr = 1e6 * max(spec.blowup_reference, 1e-30)
    store.upload_known(*marching.greville_samples(spec))
    for _ in range(args.warmup):
        store.run_resident(thr, 1)
    barrier()
    with ClockSampler(local) as clk:
        tm = store.run_resident(thr, args.steps)
        barrier()
    dev_ms = max_over_ranks(tm["total_ms"])
    value = args.steps * (nt - 1) / (dev_ms * 1e-3)
    pspec = per_step_spec(spec)  # the reference's per-step data callables
    for _ in range(max(2, args.warmup)):
        h = marching.march(pspec, mats=store)
    barrier()
    t0 = _time.perf_counter()
    e2e_steps = max(2, args.steps)
    for _ in range(e2e_steps):
        h = marching.march(pspec, mats=store)
    barrier()
    e2e = e2e_steps * (nt - 1) / max_over_ranks(_time.perf_counter() - t0)
    fp64 = C.c_double(0.0)
    _lib.check(_lib.load().tdw_fp64_peak(ctx.h, C.byref(fp64)), ctx.h, "tdw_fp64_peak")
    # roofline of the dominant kernel: the leaf level's M2L contraction (own DMMA
    # kernel), FLOPs per launch (non-dark operators) / its average launch time
    mf, m2l_ms = C.c_double(0.0), C.c_float(0.0)
    _lib.check(_lib.load().tdw_fmm_time_m2l(store.h, 10, C.byref(mf), C.byref(m2l_ms)), ctx.h,
               "tdw_fmm_time_m2l")
    achieved = max_over_ranks(mf.value / max(m2l_ms.value * 1e-3, 1e-12) / 1e12 if m2l_ms.value else 0.0)
    # whole-loop M2L rate: this rank's share of the M2L FLOPs of the loop / loop time
    loop_rate = m2l_flops(plan, nt, spec.basis.d) * info["fmm_m2l_pairs"] / max(
        1, sum(len(l.il_obs) for l in plan.levels.values())) / (dev_ms / args.steps * 1e-3) / 1e12
    try:
        ncu_m2l = json.loads((ROOT / "profiles" / "m2l_ncu.json").read_text())
    except Exception:
        ncu_m2l = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE scenario, generated meshes and incident pulse)",
            "config": {"workload": scenarios.DESCRIPTION[args.config] + ", interpolation FMM ps = pt = 4, "
                       "Z = 20, mu = 8 (corrected algorithm)", "ns": ns, "nt": nt,
                       "mot_steps_per_bench_step": nt - 1, "parallelism": f"target cells x{world}",
                       "leaf_level": plan.leaf, "m2l_pairs_this_rank": info["fmm_m2l_pairs"],
                       "near_band_entries": info["n_band"], "plan_host_s": t_plan},
            "e2e": {"value": e2e, "unit": "steps/s",
                    "h2d_bytes_per_step": sum(f is not None for f in (spec.u_data, spec.q_data)) * (nt - 1) * ns * 8,
                    "d2h_bytes_per_step": 4 * (nt - 1) * ns * 8, "api": "marching.march(spec, mats=FmmStore)"},
            "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64.value, "unit": "TFLOP/s",
                         "frac": achieved / fp64.value, "traffic": None,
                         "kernel": "m2l_dmma_kernel (own, FP64 tensor cores: mma.sync m8n8k4 f64), "
                                   "leaf level, one launch = one level tick",
                         "flops_per_launch": mf.value, "avg_launch_ms": m2l_ms.value,
                         "peak_source": "measured live (tdw_fp64_peak: DFMA chains)",
                         "ncu": ncu_m2l,
                         "whole_loop_m2l_tflops": loop_rate},
            "cpu_baseline": None, "clocks": clk.summary(), "gpu_launches": None,
        }
        print(json.dumps(line), flush=True)
    store.close()


def run_ours(args, world, rank, local):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2111_05205_b200 import _lib, distributed, marching, scenarios

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = _lib.Context(local)
    _lib.set_default_context(ctx)
    if world > 1:
        distributed.init_comm(ctx, dist)

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    spec = scenarios.build_spec(args.config)
    ns, nt = spec.mesh.n_elements, spec.nt
    thr = 1e6 * max(spec.blowup_reference, 1e-30)

    # assembly (K1 fused with the kappa combination): timed separately
    if args.fmm:
        return run_fmm(args, world, rank, local, ctx, spec, barrier, max_over_ranks)
    store = marching.BandStore(spec, nranks=world, rank=rank).assemble()
    info = store.info()
    uk, qk = marching.greville_samples(spec)
    store.upload_known(uk, qk)

    for _ in range(args.warmup):
        store.run_resident(thr, 1)
    barrier()
    with ClockSampler(local) as clk:
        tm = store.run_resident(thr, args.steps)
        barrier()
    dev_ms = max_over_ranks(tm["total_ms"])
    steps_total = args.steps * (nt - 1)
    value = steps_total / (dev_ms * 1e-3)
    # roofline pass: the same K loops with CUDA-event nodes around every K2 launch
    # (kept out of the timed pass above: the event nodes perturb the overlap)
    tk = store.run_resident(thr, args.steps, time_kernels=True)
    barrier()
    conv_ms = max_over_ranks(tk["conv_ms"] / max(tk["conv_launches"], 1))
    # the same kernel launched back to back with nothing beside it (outside the timed region)
    try:
        conv_alone_ms = store.time_conv(20)
    except Exception:
        conv_alone_ms = -1.0
    conv_alone_ms = max_over_ranks(conv_alone_ms)  # (the collective outside the try: every rank calls it)
    if conv_alone_ms <= 0.0:
        conv_alone_ms = None

    # e2e: public API with host buffers, every step, with the REFERENCE's data
    # contract: plain per-step callables u_data(t) / q_data(t), called once per
    # step in order (marching.py:258-276).  >= 2 warm-up calls: march() keeps two
    # pooled page-locked output blocks in flight
    pspec = per_step_spec(spec)
    h = None
    for _ in range(max(2, args.warmup)):
        h = marching.march(pspec, mats=store)
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(3, args.steps)
    for _ in range(e2e_steps):
        h = marching.march(pspec, mats=store)
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    e2e = e2e_steps * (nt - 1) / e2e_s
    # the scenario's own vectorised data source (PlanePulseData.sample_many: every
    # step at once on a thread pool): reported beside e2e, not as it
    for _ in range(2):
        h = marching.march(spec, mats=store)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h = marching.march(spec, mats=store)
    barrier()
    e2e_vec = e2e_steps * (nt - 1) / max_over_ranks(time.perf_counter() - t0)
    # the same call with the boundary data sampled on the device:
    # reported beside e2e, not as it (no host input copy)
    for _ in range(2):
        h = marching.march(spec, mats=store, device_data=True)
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        h = marching.march(spec, mats=store, device_data=True)
    barrier()
    e2e_dev = e2e_steps * (nt - 1) / max_over_ranks(time.perf_counter() - t0)
    # cold march(spec): a new store every call (problem setup, assembly K1, loop,
    # copies): the reference's march() rebuilds its matrices on every call too
    e2e_asm = None
    if world == 1:
        h = marching.march(pspec)
        del h
        t0 = time.perf_counter()
        n_cold = 3
        for _ in range(n_cold):
            h = marching.march(pspec)
            del h
        e2e_asm = n_cold * (nt - 1) / (time.perf_counter() - t0)
    # march() copies the samples of each data callable that is not None (pinned buffers)
    h2d = sum(f is not None for f in (spec.u_data, spec.q_data)) * (nt - 1) * ns * 8
    d2h = 4 * (nt - 1) * ns * 8

    # roofline of K2 (history convolution), algorithmic bytes = 16 B per band entry
    pk = peaks()
    peak = pk.get("hbm_gbs")
    peak_src = "measured" if peak else "fallback"
    peak = peak or HBM_FALLBACK
    n_band = max_over_ranks(float(info["n_band"]))
    kb = info["steps_per_pass"]
    # K2 roofline: the bytes one launch must move = the store read once (16 B per
    # band entry, SURVEY 8(d)'s per-step unit), over the measured launch time.
    # Temporal blocking computes kb MOT steps from that one read; that gain is
    # reported on its own (blocking), not folded into frac.
    stream = 16.0 * n_band / (conv_ms * 1e-3) / 1e9
    rpw = store.info()["conv_rpw"]  # set when the loop plan is made
    kname = f"conv_kernel_wg<{kb}>" if rpw == 4 else (
        f"conv_kernel_wg2<{kb}>" if rpw == 3 else f"conv_kernel<{kb}>")
    traffic, traffic_src = None, None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():  # ncu --set full DRAM bytes of THIS kernel at THIS kb and config
        try:
            rec = json.loads(prof.read_text()).get(f"config{args.config}")
            if rec and rec.get("kb") == kb and rec.get("n_band") == int(n_band) and world == 1:
                traffic, traffic_src = rec["dram_bytes_per_launch"], rec["source"]
        except Exception:
            traffic = None

    # roofline of K1 (coefficient fill, FP64-pipe bound): SURVEY 8(d) cost model in
    # FP64 instruction-equivalents per (i,j,gamma) evaluation, against the FP64 FMA
    # peak measured live on this GPU (tdw_fp64_peak; FMA = 2 FLOP)
    import ctypes as C
    fp64 = C.c_double(0.0)
    _lib.check(_lib.load().tdw_fp64_peak(ctx.h, C.byref(fp64)), ctx.h, "tdw_fp64_peak")
    kind = "bm" if spec.bie == "bmbie" else "uw"
    cost = K1_COST[(kind, spec.basis.d)]
    # whole-job rate: the evaluations of all ranks (each assembles only its rows) over
    # the slowest rank's fill time
    n_evals_all = info["n_evals"]
    if world > 1:
        t = torch.tensor([float(info["n_evals"])], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        n_evals_all = int(t.item())
    evals_per_s = n_evals_all / (max_over_ranks(info["t_fill_ms"]) * 1e-3)
    asm_ms = max_over_ranks(info["t_assemble_ms"])  # (collectives stay outside the rank-0 block below)
    try:  # the fill kernel's own FP64-pipe utilisation from the committed ncu capture
        k1_ncu = json.loads((ROOT / "profiles" / "k1_fill.json").read_text())
    except Exception:
        k1_ncu = None
    k1_achieved = evals_per_s * cost * 2.0 / 1e12

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_full_loop(spec)
        except Exception as exc:  # the CPU leg must not sink the GPU line
            cpu = {"value": None, "unit": "steps/s", "cores": os.cpu_count(), "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dev_ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE scenario, generated meshes and incident pulse)",
            "config": {"workload": scenarios.DESCRIPTION[args.config], "ns": ns, "nt": nt,
                       "mot_steps_per_bench_step": nt - 1, "parallelism": f"rows x{world}",
                       "l2": "banded store 1.5 GB > 126 MB L2 (no flush needed)"
                       if args.config >= 2 else "store fits in L2",
                       "gamma_star": info["gamma_star"], "n_band": int(n_band),
                       "steps_per_conv_pass": info["steps_per_pass"],
                       "solve_cluster": info["solve_cluster"], "conv_grid": info["conv_grid"]},
            "e2e": {"value": e2e, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "marching.march(spec, mats=store)",
                    "data": "plain per-step callables u_data(t) / q_data(t) (the reference's contract, "
                            "marching.py:258-276), sampled on the host every call"},
            "e2e_vectorised_data": {"value": e2e_vec, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                                    "d2h_bytes_per_step": d2h, "api": "marching.march(spec, mats=store)",
                                    "note": "the scenario's PlanePulseData.sample_many (all steps at once, "
                                            "16-thread pool) instead of per-step callables; not the e2e metric"},
            "e2e_device_boundary_data": {"value": e2e_dev, "unit": "steps/s", "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": d2h,
                                         "api": "marching.march(spec, mats=store, device_data=True)",
                                         "note": "incident-pulse samples computed on the device; not the e2e metric"},
            "e2e_with_assembly": {"value": e2e_asm, "unit": "steps/s", "api": "marching.march(spec)",
                                  "note": "every call builds the store (geometry, K1 fill, near "
                                          "structure, solver setup) and runs the loop with host data"},
            "roofline": {"bound": "hbm", "achieved": stream, "peak": peak, "unit": "GB/s",
                         "frac": stream / peak, "traffic": traffic, "kernel": f"{kname} (K2, history convolution)",
                         "peak_source": peak_src, "avg_launch_ms": conv_ms,
                         "launches_timed": int(tk["conv_launches"]),
                         "bytes_per_launch": 16.0 * n_band,
                         "traffic_source": traffic_src,
                         "traffic_over_algorithmic": (traffic / (16.0 * n_band)) if traffic else None,
                         "kernel_alone": ({"avg_launch_ms": conv_alone_ms,
                                           "achieved": 16.0 * n_band / (conv_alone_ms * 1e-3) / 1e9,
                                           "frac": 16.0 * n_band / (conv_alone_ms * 1e-3) / 1e9 / peak,
                                           "note": "20 launches back to back with nothing beside them; "
                                                   "achieved / frac above are the launches INSIDE the timed "
                                                   "loops, where the solve cluster and the near steps run "
                                                   "beside the pass"} if conv_alone_ms else None),
                         "note": "algorithmic bytes per launch = 16 B x N_band (V_U, V_W fp64, the "
                                 "store read once); a launch computes kb MOT steps from that read "
                                 "(see blocking)"},
            "blocking": {"steps_per_launch": kb,
                         "survey_unit_GBps": 16.0 * n_band * kb / (conv_ms * 1e-3) / 1e9,
                         "note": "SURVEY 8(d) counts 16 B x N_band per MOT step; temporal blocking "
                                 "serves kb steps per store read, so this rate is kb x the "
                                 "physical stream and is not an HBM fraction"},
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            # per loop: init_hist + (conv_kernel + reduce_parts) per pass + (solve +
            # near_step) per step
            "gpu_launches": int(args.steps * (1 + 2 * (-(-(nt - 1) // info["steps_per_pass"])) + 2 * (nt - 1))),
            "assembly": {"ms": asm_ms, "evals": n_evals_all,
                         "evals_per_s": evals_per_s,
                         "metric": "(i,j,gamma) layer-potential evals/s (fill kernel, fp64)",
                         "roofline": {"bound": "fp64",
                                      "frac": k1_ncu.get("fp64_pipe_active") if k1_ncu else None,
                                      "achieved": (k1_ncu["fp64_pipe_active"] * fp64.value) if k1_ncu else None,
                                      "peak": fp64.value, "unit": "TFLOP/s",
                                      "kernel": "fill_kernel (K1)",
                                      "source": "ncu sm__pipe_fp64_cycles_active of the fill kernel at "
                                                "this configuration (profiles/k1_fill.json)",
                                      "peak_source": "measured live (tdw_fp64_peak: DFMA chains)",
                                      "ncu": k1_ncu},
                         "cost_model_rate": {"tflops_equiv": k1_achieved, "cost_per_eval": cost,
                                             "note": "SURVEY 8(d): FP64 instruction-equivalents per "
                                                     "evaluation (div/sqrt 20, atan 26, asinh 60); "
                                                     "hoisting raises evals/s while the cost stays "
                                                     "fixed, so this is not a pipe fraction"}},
            "graph": bool(tm.get("solve_ms", 0) > 0),
        }
        print(json.dumps(line), flush=True)
    store.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--ref-chunk", type=int, default=0,
                    help="MOT steps per reference-arm bench step (default (nt-1)/8)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--fmm", action="store_true", help="interpolation FMM path (configs 3-4; default for 4)")
    args = ap.parse_args()
    if args.config == 4:
        args.fmm = True  # the direct store of config 4 is ~200 GB
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
