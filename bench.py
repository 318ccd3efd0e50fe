#!/usr/bin/env python
"""Benchmark of the periscat hot path on B200 (driver contract).

Step   = one S-preconditioned Schur matvec  y = v - S (T v - B A^+ C v)  on
         BASELINE.json configs[2] (cfg3: M=1000 inclusions, p=25, 1 RHS):
         K3 (C) -> K4 (A^+) -> K5 (B) -> K1 (all-pairs M2L, 2,999,000
         translations) -> epilogue.  Multi-GPU: target inclusions sharded,
         v all-gathered over NCCL, C partial sums all-reduced.
value  = inclusion-pair translations per second over the whole job.
e2e    = same metric through the public operator call SchurOperator.__call__
         (what solver.apply_schur_operator runs), with v copied H2D from a
         pinned host buffer and y copied D2H into one inside the timed region.
Also reported: M=1000 full-solve seconds (the metric's second half), the K1
roofline against the box's measured FP64 peak (max of the DFMA and DMMA chain
microbenchmarks), and the CPU oracle baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import os

for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse
import ctypes
import json
import math
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
import workloads  # noqa: E402

METRIC = "inclusion-pair translations/s (FP64 % peak) and M=1000 full-solve seconds"
UNIT = "translations/s"
CFG = 3


def _config_block(cfg_id, M, p, nrhs, world, decomposition="targets"):
    return {"workload": f"cfg{cfg_id}: S-preconditioned Schur matvec, M={M} inclusions, p={p} "
                        f"(L={2 * p + 1}), {nrhs} RHS, 3-layer grating omega=10, "
                        "theta_ref=-7pi/10, P=1 near-field copies",
            "M": M, "p": p, "nrhs": nrhs, "translations_per_step": M * (3 * M - 1) * nrhs,
            "parallelism": (f"tile-pair-sharded x{world} (symmetric K1s + reduce-scatter)"
                            if decomposition == "pairs" else f"target-sharded x{world}"),
            "coupling": "pre-assembled C^T / B_phys (device GEMVs)",
            "l2": "flushed (256 MiB write) before every timed step"}


# ----------------------------------------------------------------------------- CPU baseline
_POOL_STATE = {}


def _pool_init(beta, centers, k2, p, bloch):
    _POOL_STATE.update(beta=beta, centers=centers, k2=k2, p=p, bloch=bloch)


def _pool_work(targets):
    from oracle import periscat_oracle as O
    s = _POOL_STATE
    t0 = time.perf_counter()
    O.apply_T(s["beta"], s["centers"], s["k2"], s["p"], s["bloch"], targets=targets)
    return time.perf_counter() - t0


def cpu_oracle_rate(steps: int, warmup: int, per_worker: int = 12):
    """The oracle's apply_T (NumPy restatement of multiscat.apply_T)
    on a bounded target sample, one process per host core.  Returns
    (translations/s, cores, sample description, per-step seconds)."""
    import multiprocessing as mp
    from oracle import periscat_oracle as O
    pb = O.load_problem(CFG)
    cores = len(os.sched_getaffinity(0))
    rng = np.random.default_rng(0)
    beta = pb.smat[None, :] * (rng.standard_normal((pb.M, pb.L)) + 1j * rng.standard_normal((pb.M, pb.L)))
    ntarget = cores * per_worker
    tids = np.arange(ntarget) % pb.M
    chunks = [tids[i::cores] for i in range(cores)]
    # spawn, not fork: on the GPU arm this runs after CUDA / NCCL threads exist
    ctx = mp.get_context("spawn")
    times = []
    with ctx.Pool(cores, initializer=_pool_init,
                  initargs=(beta, pb.centers, pb.es.k2, pb.p, pb.es.bloch)) as pool:
        for it in range(warmup + steps):
            t0 = time.perf_counter()
            pool.map(_pool_work, chunks)
            dt = time.perf_counter() - t0
            if it >= warmup:
                times.append(dt)
    tr = ntarget * (3 * pb.M - 1)
    rate = tr / float(np.mean(times))
    sample = (f"oracle apply_T (NumPy, SPEC.md:504 restated), {ntarget} target inclusions x "
              f"{3 * pb.M - 1} source images of cfg{CFG} per step ({tr} translations), "
              f"{cores} processes x 1 BLAS thread; C/B/A^+ (~5% of CPU time) not included")
    return rate, cores, sample, times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    rate, cores, sample, times = cpu_oracle_rate(args.steps, args.warmup)
    from oracle import periscat_oracle as O
    pb = O.load_problem(CFG)
    line = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(times) * 1e3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)",
            "data": "synthetic (seeded reference geometry fixture)",
            "config": _config_block(CFG, pb.M, pb.p, 1, 1),
            "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": sample},
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi in loop mode (-lms 100) for the duration of the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                self.out = ""

    def summary(self):
        rows = [[x.strip() for x in ln.split(",")] for ln in self.out.strip().splitlines() if ln]
        rows = [r for r in rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in rows) if v is not None]
        pw = [v for v in (num(r[2]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[3 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(rows)}


def _guarded(fn, world):
    """Run an auxiliary measurement block; on one GPU a failure is recorded in
    the JSON line instead of losing the headline (with several ranks an
    exception must propagate: a rank leaving a collective would hang the rest)."""
    if world > 1:
        return fn()
    try:
        return fn()
    except Exception as e:   # noqa: BLE001 -- reported, not swallowed
        import traceback
        traceback.print_exc(file=sys.stderr)
        return {"error": f"{type(e).__name__}: {e}"}


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_1412_7466_b200 import _lib, grating, parallel, solver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # PS_BENCH_ONE_GPU=1 + PS_BENCH_BACKEND=gloo: every rank on cuda:0 over
    # gloo -- exercises the multi-rank bench path on a one-GPU box (timings
    # meaningless); the driver's runs use one GPU per rank over NCCL
    if os.environ.get("PS_BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("PS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    lib = _lib.load()
    peak = ctypes.c_double()
    pms = ctypes.c_double()
    _lib.check(None, lib.ps_dfma_peak(local, ctypes.byref(peak), ctypes.byref(pms)))
    tpeak = ctypes.c_double()
    _lib.check(None, lib.ps_dmma_peak(local, ctypes.byref(tpeak)))

    sysm, centers, p, radius = workloads.load_config(CFG)
    M, L = centers.shape[0], 2 * p + 1
    t0, t1 = (M * rank) // world, (M * (rank + 1)) // world
    op = solver.SchurOperator(sysm, centers, p, radius=radius, device=local,
                              target_range=(t0, t1))
    eng = op.eng
    rng = np.random.default_rng(1234)
    v_host = op.smat[None, None, :] * (rng.standard_normal((1, M, L)) + 1j * rng.standard_normal((1, M, L)))
    v_full = torch.as_tensor(v_host).to(dev).contiguous()
    v_own = v_full[:, t0:t1].contiguous()
    y = eng.empty_own()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    # one Schur matvec: N=1 -> the operator on the resident full vector;
    # N>1 -> parallel.ShardedSchur (NCCL all-gather of beta, C partial over own
    # sources + all-reduce, own-target B/S; the M2L either over all sources for
    # the own targets or, while M / N >= 200, the symmetric K1s over 1/N of the
    # tile pairs + NCCL reduce-scatter) -- the path gmres_dist drives
    sharded = parallel.ShardedSchur(op) if world > 1 else None

    def step():
        if world == 1:
            op(v_full, out=y)
        else:
            sharded(v_own, out=y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.stats_reset()
    eng.profile(True)
    st = torch.cuda.current_stream()
    tot = 0.0
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)                      # evict L2 (126 MB) between timed steps
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            step()
            e1.record(st)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    eng.profile(False)
    stats = eng.stats()
    tmax = torch.tensor([tot], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms_step = float(tmax.item()) / args.steps
    tr_step = M * (3 * M - 1)
    value = tr_step / (ms_step * 1e-3)

    # K1 roofline (this rank's own launches; algorithmic flops = 8 L^2 per translation)
    fp64_peak = max(peak.value, tpeak.value)
    k1_avg_ms = stats["k1_ms"] / max(stats["k1_count"], 1)
    k1_flops = (t1 - t0) * (3 * M - 1) * 8.0 * L * L
    achieved = k1_flops / (k1_avg_ms * 1e-3) / 1e12
    traffic = None
    tf = os.path.join(ROOT, "profiles", "k1_dram_bytes.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"cfg{CFG}")
        except Exception:
            traffic = None

    # e2e through the public API with pinned host buffers (N=1: full call;
    # N>1: every rank's call, max over ranks)
    vh = torch.as_tensor(v_host if world == 1 else v_host[:, t0:t1]).contiguous().pin_memory()
    yh = torch.empty((1, t1 - t0, L), dtype=torch.complex128).pin_memory()

    def e2e_step():
        vd = vh.to(dev, non_blocking=True)
        if world == 1:
            op(vd, out=y)
        else:
            sharded(vd, out=y)
        yh.copy_(y, non_blocking=True)

    for _ in range(max(args.warmup, 1)):
        e2e_step()
    torch.cuda.synchronize()
    te = 0.0
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        e2e_step()
        e1.record(st)
        e1.synchronize()
        te += e0.elapsed_time(e1)
    temax = torch.tensor([te], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(temax, op=dist.ReduceOp.MAX)
    e2e_value = tr_step / (float(temax.item()) / args.steps * 1e-3)

    # full solve (M=1000): setup + GMRES to 1e-10 + recovery.  N=1: device
    # GMRES (ps_gmres); N>1: parallel.gmres_dist over the sharded operator
    # (NCCL all-gather of each Krylov vector, all-reduced dot products).
    # Starts from the grating config: the empty-grating matrix is assembled and
    # factorised on the device (ps_setup_empty), as solve_full(config) does.
    conf = sysm.config

    def full_solve(diagnostics=False):
        if world == 1:
            return solver.solve_full(conf, centers, p, radius=radius, device=local,
                                     diagnostics=diagnostics)
        opd = solver.SchurOperator(conf, centers, p, radius=radius, device=local,
                                   target_range=(t0, t1), split_setup=True)
        sh = parallel.ShardedSchur(opd)
        x, its, hist = parallel.gmres_dist(sh, sh.rhs(), 1e-10, 150, engine=opd.eng)
        xe = sh.recover(x.contiguous())
        c, d = opd.split_cd(xe)
        from paper_1412_7466_b200 import postproc
        fl = postproc.flux_error(c[0], d[0], sysm.config)
        a_ms, s_ms = opd.eng.setup_timings()
        return solver.Solution(None, c, d, its, hist, [fl],
                               dict(assemble_ms=a_ms, svd_ms=s_ms))

    def timed_full_solve():
        def timed():
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            ts = time.perf_counter()
            sol = full_solve()
            torch.cuda.synchronize()
            tsol = torch.tensor([time.perf_counter() - ts], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(tsol, op=dist.ReduceOp.MAX)
            return sol, float(tsol.item())
        _, cold = timed()                           # first call: lazy cuSOLVER / module loads
        sol, warm = timed()
        diag = full_solve(diagnostics=True) if world == 1 else None
        return {"seconds": warm, "cold_seconds": cold, "iterations": sol.iterations[0],
                "coupled_residual": diag.coupled_residual[0] if diag else None,
                "wall_residual": diag.wall_residual[0] if diag else None,
                "flux_error": sol.flux[0]["error"],
                "driver": "ps_gmres (device)" if world == 1 else "parallel.gmres_dist (NCCL)",
                "setup_device_ms": {"empty_assembly": sol.timings.get("assemble_ms"),
                                    "svd_and_pinv_factors": sol.timings.get("svd_ms")},
                "note": "wall clock from the grating config and the inclusion centres: device "
                        "assembly of the 856x781 empty-grating matrix, cuSOLVER SVD, operator "
                        "setup (S, geometry, coupling blocks), GMRES to 1e-10 and recovery; "
                        "max over ranks; 'seconds' is the warm (second) call, 'cold_seconds' "
                        "the first; the residuals (SPEC.md:571 coupled system, eg:396-433 wall "
                        "discrepancy) come from a third, untimed call"}

    full = _guarded(timed_full_solve, world)

    # the other BASELINE configs that fit one step (cfg1 M=10, cfg2 M=100, cfg4
    # Wood anomaly M=1000): one Schur matvec and solve_full(config) each
    others = None
    if world == 1 and not args.no_cfg5:
        others = _guarded(lambda: other_configs(local), world)

    # cfg5 (M=1e4, p=20, 16 incidence angles): the multi-RHS K1 alone, own
    # target shard, translations/s over the whole job, K1m roofline
    cfg5 = None
    if not args.no_cfg5:
        sus = ctypes.c_double()
        _lib.check(None, lib.ps_dfma_sustained(local, 3.0, ctypes.byref(sus)))
        cfg5 = _guarded(lambda: cfg5_apply_T(dev, local, rank, world, sus.value, tpeak.value,
                                             args), world)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        def cpu_leg():
            rate, cores, sample, _ = cpu_oracle_rate(3, 1)
            return {"value": rate, "unit": UNIT, "cores": cores, "kind": "port",
                    "sample": sample}
        cpu = _guarded(cpu_leg, world)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "c128 (f64)", "data": "synthetic (seeded reference geometry fixture)",
                "config": _config_block(CFG, M, p, 1, world,
                                        sharded.mode if sharded is not None else "targets"),
                "roofline": {"bound": "fp64", "achieved": achieved, "peak": fp64_peak,
                             "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                             "traffic": traffic,
                             "kernel": "m2l_sym_stage_kernel (K1s, symmetric single-RHS M2L fed by "
                                       "the symbol store, coefficient rows staged in shared "
                                       "memory; m2l_sym_kernel when the store does not fit)"
                                       if world == 1 or sharded.mode == "pairs"
                                       else "m2l_kernel (K1, tiled; target shard)",
                             "k1_avg_ms": k1_avg_ms,
                             "algorithmic": "8(2p+1)^2 flops per translation",
                             "executed": "Karatsuba complex MACs: 3 real FMA (6 flops) per "
                                         "complex MAC, i.e. 6(2p+1)^2 FP64 flops issued per "
                                         "translation; the geometry-only translation symbols "
                                         "come from the precomputed symbol store (TMA bulk "
                                         "copies; generated in the kernel when the store does "
                                         "not fit); the DFMA sweeps carry operand-reuse "
                                         "flags set post-link (sass_reuse_patch.py); "
                                         "'achieved' counts the 8(2p+1)^2 algorithmic flops",
                             "peak_source": "max of the two FP64 chain microbenchmarks measured on "
                                            "this GPU in this run (MEASURED_PEAKS.json has no FP64 "
                                            "entry): ps_dfma_peak (DFMA chains, 8 CTAs/SM) and "
                                            "ps_dmma_peak (mma.sync f64 chains); both pipes are "
                                            "one unit on B200 (tools/fp64_pipes.cu: mixed "
                                            "DFMA+DMMA warps sum to the same 36.8 TF/s); nominal "
                                            "148 SM x 64 FMA x 2 x 1.965 GHz = 37.2 TF/s",
                             "dfma_chain_peak": peak.value,
                             "dmma_chain_peak": tpeak.value,
                             "frac_of_dfma_chain": achieved / peak.value},
                "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": UNIT,
                        "h2d_bytes_per_step": int(vh.numel() * 16),
                        "d2h_bytes_per_step": int(yh.numel() * 16)},
                "gpu_launches": int(stats["launches"]),
                "clocks": clk.summary(),
                "full_solve_m1000": full,
                "other_configs": others,
                "cfg5_apply_T_16rhs": cfg5}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def other_configs(local):
    """cfg1 / cfg2 / cfg4 (BASELINE configs[0, 1, 3]): Schur matvec time and
    warm solve_full(config) seconds with iterations and flux error."""
    import torch

    from paper_1412_7466_b200 import grating, solver
    out = {}
    for cfg in (1, 2, 4):
        sysm, centers, p, radius = workloads.load_config(cfg)
        conf = sysm.config
        M, L = centers.shape[0], 2 * p + 1
        op = solver.SchurOperator(conf, centers, p, radius=radius, device=local)
        rng = np.random.default_rng(cfg)
        v = torch.as_tensor(op.smat[None, None, :] * (rng.standard_normal((1, M, L))
                            + 1j * rng.standard_normal((1, M, L)))).cuda()
        y = torch.empty_like(v)
        for _ in range(3):
            op(v, out=y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            op(v, out=y)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / n
        solver.solve_full(conf, centers, p, radius=radius, device=local, diagnostics=False)   # warm
        torch.cuda.synchronize()
        t = time.perf_counter()
        sol = solver.solve_full(conf, centers, p, radius=radius, device=local, diagnostics=False)
        torch.cuda.synchronize()
        out[f"cfg{cfg}"] = {"M": M, "p": p, "matvec_ms": ms,
                            "translations_per_s": M * (3 * M - 1) / (ms * 1e-3),
                            "full_solve_seconds": time.perf_counter() - t,
                            "iterations": sol.iterations[0],
                            "flux_error": sol.flux[0]["error"]}
        del op
    return out


def cfg5_apply_T(dev, local, rank, world, dfma_peak, tensor_peak, args):
    import torch
    import torch.distributed as dist

    from paper_1412_7466_b200.engine import Engine
    centers = np.load(os.path.join(ROOT, "tests", "golden", "centers_cfg5.npy"))
    M, p, R = centers.shape[0], 20, 16
    L = 2 * p + 1
    th = np.linspace(-math.pi / 3, math.pi / 3, R) - math.pi / 2
    eng = Engine(local)
    eng.set_geometry(centers, p, 12.0, 1.0, 1)
    eng.set_bloch(np.exp(1j * 10.0 * np.cos(th)))
    t0, t1 = (M * rank) // world, (M * (rank + 1)) // world
    eng.set_target_range(t0, t1)
    rng = np.random.default_rng(5)
    v = torch.as_tensor(rng.standard_normal((R, M, L)) + 1j * rng.standard_normal((R, M, L))).to(dev)
    out = eng.empty_own()
    eng.apply_T(v, out)                       # warm-up (also sizes the workspaces)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    eng.stats_reset()
    eng.profile(True)
    steps = max(1, min(args.steps, 3))
    st = torch.cuda.current_stream()
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            eng.apply_T(v, out)
        e1.record(st)
        e1.synchronize()
    eng.profile(False)
    stats = eng.stats()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    tr = M * (3 * M - 1) * R
    k1_ms = stats["k1_ms"] / max(stats["k1_count"], 1)
    flops = (t1 - t0) * (3 * M - 1) * R * 8.0 * L * L
    ach = flops / (k1_ms * 1e-3) / 1e12
    eng.close()
    return {"workload": f"cfg5: apply_T, M={M}, p={p}, {R} RHS (incidence angles), "
                        "target-sharded", "ms_per_step": ms, "steps": steps,
            "value": tr / (ms * 1e-3), "unit": UNIT,
            "roofline": {"bound": "fp64", "achieved": ach, "peak": tensor_peak,
                         "unit": "TFLOP/s", "frac": ach / tensor_peak,
                         "kernel": "m2l_mma_kernel (K1d: mma.sync m8n8k4 f64 FP64 tensor cores)",
                         "executed": "Karatsuba: 3 real MMAs per complex tile (6L^2 issued vs 8L^2 algorithmic flops per translation)",
                         "peak_source": "ps_dmma_peak: mma.sync f64 chains on this GPU",
                         "dfma_sustained_peak": dfma_peak,
                         "frac_of_dfma_peak": ach / dfma_peak},
            "gpu_launches": int(stats["launches"]), "clocks": clk.summary()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline leg")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 16-RHS apply_T block")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
