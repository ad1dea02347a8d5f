"""Benchmark of the solve phase: Schwarz-PCG DOF*iterations/s on B200.

One "step" = one complete PCG solve  A x = f  to ||r|| <= 1e-8 ||f|| with the
two-level additive Schwarz preconditioner M_AS,2 (SNK + GenEO coarse space,
PAPER.md eq. 2.4 / §3 final display) -- every kernel of the hot path runs in
libmaxwell_dd.so.  The one-time setup (assembly, local factorisations, GenEO
GEVPs, E) runs on the device before the timed region and is reported
separately under "setup_s".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1] [--impl b200|reference]

N = 1: BASELINE.json configs[4] at one GPU (c4: 64^3 cubes x 6 tets, 4^3
subdomains, 1.8M dofs, 20k GenEO vectors) -- the largest single-GPU config
(c3, 96^3 / 512 subdomains, is the 8-GPU mesh); --config c1 / c2 for the others.
N > 1 (torchrun, one rank per GPU): every rank solves its own replica of the
workload (weak scaling, no data-path collective: the sharded solve of sharded.cu
replicates the setup and the coarse factor, so c4_weak64_xN does not fit it --
DESIGN.md §9), value = all ranks' DOF*iterations / max-over-ranks time.

--mode sharded: ONE copy of the workload with its subdomains sharded over the N
ranks (strong scaling; halo exchanges and allreduces over NCCL, mdd_shard_solve);
opt-in because no multi-GPU box was available to validate it beyond one rank.

--impl reference times the CPU oracle (oracle/, fp64 numpy/scipy) on a bounded
sample of the same recipe on rank 0; other ranks exit 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "Schwarz-PCG DOF*iterations/s"
UNIT = "DOF*iter/s"
TOL = 1e-8
# the oracle sample: the c1 recipe (channels, contrast 1e4, gamma 1e-4, overlap 1,
# threshold 0.1) on a 12^3 grid with 2^3 subdomains (setup untimed)
# the oracle sample per recipe: the same coefficients / gamma / overlap / threshold on a
# grid the oracle's dense GEVPs finish in seconds (setup untimed)
CPU_SAMPLES = {"c1": dict(n=12, p=2), "c2": dict(n=12, p=2, hole=2), "c3": dict(n=12, p=2),
               "c4": dict(m=12, q=2)}


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # c4 at N = 1 (64^3 cubes, 4^3 subdomains, 1.8M dofs): the largest single-GPU
    # configuration of BASELINE.json (c3 is the 8-GPU mesh)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # as2_coarse_start: M_AS,2 (eq. 2.4) with PCG started from x0 = Q f, one coarse
    # solve per iteration (reading R13); as2: the same operator from x0 = 0
    ap.add_argument("--variant", default="as2_coarse_start",
                    choices=["as2_coarse_start", "as2", "additive", "as1"])
    ap.add_argument("--maxit", type=int, default=2000)
    # replicas: every rank its own copy of the workload (weak scaling, the default);
    # sharded: ONE copy of the workload, its subdomains sharded over the ranks (strong
    # scaling): halo exchanges and the pTq / |r|^2 / rTz / coarse allreduces over NCCL
    # (sharded.cu); the setup is replicated on every rank
    ap.add_argument("--mode", default="replicas", choices=["replicas", "sharded"])
    return ap.parse_args()


# ------------------------------------------------------------------ clocks
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def cpu_oracle_sample(cfg, max_seconds=30.0, min_solves=1, variant="as2_coarse_start"):
    """Time the CPU oracle's solve phase (PCG to 1e-8 with M_AS,2) on the bounded
    sample; returns (DOF*iter/s, description, cores)."""
    import threadpoolctl  # noqa: F401  (scipy/numpy BLAS pools are used as they stand)
    from oracle import solver as osolver
    w = workloads.make(cfg, **CPU_SAMPLES.get(cfg, {}))
    t0 = time.perf_counter()
    P = osolver.Problem(w, variant="as2" if variant == "as2_coarse_start" else variant)
    x0 = "coarse" if variant == "as2_coarse_start" else "zero"
    setup = time.perf_counter() - t0
    f = workloads.rhs(P.n, w.f_seed)
    work, el, solves = 0.0, 0.0, 0
    while solves < min_solves or el < max_seconds * 0.3:
        t0 = time.perf_counter()
        _, it, _ = P.solve(f, tol=TOL, x0=x0)
        el += time.perf_counter() - t0
        work += P.n * it
        solves += 1
        if el > max_seconds:
            break
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    desc = (f"oracle (numpy/scipy fp64) PCG solve phase on the {cfg} recipe at "
            f"{w.nx}^3 cubes, {w.px}^3 subdomains (n={P.n}, {it} iterations, variant {variant}), "
            f"{solves} solve(s); "
            f"oracle setup {setup:.1f}s untimed")
    return work / el, desc, cores, el / solves


def run_reference(args, rank, world):
    if rank != 0:
        return
    cfg = args.config
    vals = []
    desc = cores = None
    for k in range(args.warmup + args.steps):
        v, desc, cores, _ = cpu_oracle_sample(cfg, max_seconds=10.0, variant=args.variant)
        if k >= args.warmup:
            vals.append(v)
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": None, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg + "_oracle_sample", "recipe": cfg, **CPU_SAMPLES.get(cfg, {})},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def reduce_over_ranks(ms, work, world, device):
    """Whole-job aggregation: the slowest rank's time (max) and every rank's work
    (sum).  Ranks solve independent replicas (no data-path collective); this is
    the only collective of the bench."""
    if world <= 1:
        return float(ms), float(work)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    w = torch.tensor([float(work)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(w, op=dist.ReduceOp.SUM)
    return float(t[0]), float(w[0])


def main():
    args = parse()
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2311_18783_b200 import MaxwellDD

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if args.mode == "sharded":
        run_sharded(args, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return

    w = workloads.make(args.config)
    t0 = time.perf_counter()
    G = MaxwellDD(w, device=local, variant=args.variant)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    G.set_stream(stream)
    n = G.n
    f_host = workloads.rhs(n, w.f_seed + rank)
    f = torch.as_tensor(f_host, device="cuda")
    x = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def l2_flush():
        with torch.cuda.stream(stream):
            flush.fill_(1.0)

    # ---- warm-up
    iters = []
    for _ in range(args.warmup):
        l2_flush()
        it, relres, ok = G.solve(f, x, tol=TOL, maxit=args.maxit)
        assert ok, f"PCG did not converge (relres {relres})"
        iters.append(it)

    # ---- timed steps: the whole solve is one CUDA-graph launch (device-side WHILE
    # loop); CUDA events on the library's stream, L2 flushed between steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    sw0 = G.sweep_timing("local")
    cw0 = G.sweep_timing("coarse") if G.info["n0"] else (0.0, 0)
    t_ms = 0.0
    launches = 0
    work = 0
    for _ in range(args.steps):
        l2_flush()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        it, relres, ok = G.solve(f, x, tol=TOL, maxit=args.maxit)
        e1.record(stream)
        e1.synchronize()
        assert ok
        t_ms += e0.elapsed_time(e1)
        launches += G.last_launches()
        work += n * it
        iters.append(it)
    torch.cuda.synchronize()
    sw1 = G.sweep_timing("local")
    cw1 = G.sweep_timing("coarse") if G.info["n0"] else (0.0, 0)
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    step_ms = t_ms / args.steps
    step_ms_max, total_work = reduce_over_ranks(step_ms, work, world, "cuda")
    value = total_work / (step_ms_max * args.steps / 1e3)
    in_step = ((sw1[0] - sw0[0]) / max(1, sw1[1] - sw0[1]), sw1[1] - sw0[1])
    cin_step = ((cw1[0] - cw0[0]) / max(1, cw1[1] - cw0[1]), cw1[1] - cw0[1])

    # ---- the two persistent sweeps alone (one k_sweep launch each): the local
    # solves (mdd_apply_local) and the coarse solve E^{-1} (mdd_apply_coarse_inverse),
    # CUDA events on their stream
    def timed(fn, reps=10):
        for _ in range(2):
            fn()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        e1.synchronize()
        return e0.elapsed_time(e1) / reps
    v = torch.randn(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(v)
    sweep_ms = timed(lambda: G.apply_local(v, y))
    n0 = int(G.info["n0"])
    v0 = torch.randn(max(n0, 1), dtype=torch.float64, device="cuda")
    y0 = torch.empty_like(v0)
    csweep_ms = timed(lambda: G.apply_coarse_inverse(v0, y0)) if n0 else None
    csw1 = G.sweep_timing("coarse") if n0 else None
    # per-phase breakdown of one solve (eager path with events; not the timed path)
    G.set_profiling(True)
    G.solve(f, x, tol=TOL, maxit=args.maxit)
    prof = G.profile()
    G.set_profiling(False)

    # ---- e2e: host buffers through mdd_solve_host (H2D of f + D2H of x inside)
    fp = torch.empty(n, dtype=torch.float64, pin_memory=True)
    fp.numpy()[:] = f_host
    xp = torch.empty(n, dtype=torch.float64, pin_memory=True)
    e2e_ms, e2e_work = 0.0, 0
    for _ in range(max(1, args.steps)):
        l2_flush()
        stream.synchronize()
        t0 = time.perf_counter()
        _, it, _ = G.solve_host_into(fp.numpy(), xp.numpy(), tol=TOL, maxit=args.maxit)
        e2e_ms += (time.perf_counter() - t0) * 1e3
        e2e_work += n * it
    e2e_ms_max, e2e_total = reduce_over_ranks(e2e_ms, e2e_work, world, "cuda")
    e2e_val = e2e_total / (e2e_ms_max / 1e3)

    # ---- the literal eq. (2.4) loop from x0 = 0 beside it (same handle; context)
    alt = None
    if args.variant == "as2_coarse_start":
        G.set_variant("as2")
        G.solve(f, x, tol=TOL, maxit=args.maxit)
        a_ms, a_it = 0.0, 0
        for _ in range(2):
            l2_flush()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            a_it, _, _ = G.solve(f, x, tol=TOL, maxit=args.maxit)
            e1.record(stream)
            e1.synchronize()
            a_ms += e0.elapsed_time(e1)
        a_ms /= 2
        alt = {"variant": "as2 (x0 = 0, two coarse solves per iteration)", "iterations": a_it,
               "ms_per_step": a_ms, "value": n * a_it / (a_ms / 1e3)}
        G.set_variant(args.variant)

    info = G._info()   # after the solves: kernels per iteration, launches
    roof = roofline(G, sweep_ms, in_step, csweep_ms, cin_step, t_ms, cfg=args.config)
    # the whole PCG iteration against the same roofline: algorithmic bytes of one
    # iteration (MaxwellDD.bytes_model) x iterations / device time
    bm = G.bytes_model()
    it_gbs = bm["iteration"] * iters[-1] / (step_ms / 1e3) / 1e9
    roof["iteration"] = {"bytes_per_iteration": bm["iteration"], "achieved": it_gbs,
                         "frac": it_gbs / roof["peak"], "breakdown_bytes": bm}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n_dofs": n, "subdomains": info["nsub"],
                   "n0_coarse": info["n0"], "geneo_vectors": info["ngeneo"],
                   "iterations": iters[-1], "tol": TOL, "gamma": w.gamma,
                   "variant": args.variant,
                   "parallelism": f"replicas x{world}" if world > 1 else "1 GPU",
                   "l2": "flushed between steps (256 MB write)"},
        "iterations": iters[-1],
        "sizes": info,
        "setup_s": setup_s,
        "setup_phases_s": G.setup_times(),
        "phase_ms_one_solve_eager": {k: v[0] for k, v in prof.items()},
        "variant_x0_zero": alt,
        "roofline": roof,
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches,
        "kernels_per_iteration": int(info.get("kernels_per_iter", 0)),
        "clocks": clocks,
        "paper_context": ("PAPER.md §4 (FreeFEM/PETSc GMRES on CPUs, hexahedral beam meshes): "
                          "AS-SNK-GenEO takes 23-28 iterations across Tables 3-7; ~300 GenEO "
                          "vectors per subdomain in the mu_alt = 1e4 case (Table 5); context only"),
    }
    if rank == 0 and not args.no_cpu_baseline:
        v, desc, cores, _ = cpu_oracle_sample(args.config, variant=args.variant)
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": desc}
    if rank == 0:
        print(json.dumps(line), flush=True)
    G.close()
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, rank, world, local):
    """One copy of the workload, its subdomains sharded over the ranks (strong
    scaling; mdd_shard_setup / mdd_shard_solve): per iteration the forward halos of
    p, r and w, the reverse halo of the local solves, the allreduces of pTq, |r|^2,
    rTz, Z^T r and the two exchanges of the distributed coarse solve go over NCCL.
    The setup (and E's factor, swept by subtree) is replicated on every rank.
    value = n * iterations / max-over-ranks device time."""
    import torch
    import torch.distributed as dist
    from paper_2311_18783_b200 import MaxwellDD

    w = workloads.make(args.config)
    t0 = time.perf_counter()
    G = MaxwellDD(w, device=local, variant=args.variant)
    sh = G.shard_setup(rank, world)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.Stream()
    G.set_stream(stream)
    uid = [bytes(torch.cuda.nccl.unique_id()) if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    G.shard_nccl_init(uid[0])
    n, n_own = G.n, sh["n_own"]
    f_host = workloads.rhs(n, w.f_seed)[G.owned]
    f = torch.as_tensor(f_host, device="cuda")
    x = torch.empty(n_own, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def step(host=False):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        it, relres, ok = G.shard_solve(f, x, tol=TOL, maxit=args.maxit)
        e1.record(stream)
        e1.synchronize()
        assert ok, f"sharded PCG did not converge (relres {relres})"
        return e0.elapsed_time(e1), it

    for _ in range(args.warmup):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk = Clocks(local)
    clk.start()
    t_ms, it = 0.0, 0
    for _ in range(args.steps):
        ms, it = step()
        t_ms += ms
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    step_ms = t_ms / args.steps
    # every rank reports the same iterations; the job's work is n * it once
    step_ms_max, _ = reduce_over_ranks(step_ms, 0.0, world, "cuda")
    value = n * it / (step_ms_max / 1e3)
    # e2e: this rank's part of f from pinned host memory, its part of x back
    import ctypes as C
    from paper_2311_18783_b200 import _lib as L
    fp = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
    fp.numpy()[:] = f_host
    xp = torch.empty(n_own, dtype=torch.float64, pin_memory=True)
    e2e_ms = 0.0
    for _ in range(max(1, args.steps)):
        with torch.cuda.stream(stream):
            flush.fill_(1.0)
        stream.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        itc, rel = C.c_int(0), C.c_double(0.0)
        rc = L.lib().mdd_shard_solve(G._h, fp.data_ptr(), xp.data_ptr(), TOL, args.maxit, 1,
                                     C.byref(itc), C.byref(rel))
        assert rc == L.MDD_OK, rc
        e2e_ms += (time.perf_counter() - t0) * 1e3
    e2e_ms_max, _ = reduce_over_ranks(e2e_ms / max(1, args.steps), 0.0, world, "cuda")
    info = G._info()
    peak, src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    # the whole job's algorithmic bytes per iteration (the single-GPU model: the
    # replicated top of E is counted once) against world x the measured HBM peak
    bm = G.bytes_model()
    gbs = bm["iteration"] * it / (step_ms_max / 1e3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n_dofs": n, "subdomains": info["nsub"], "n0_coarse": info["n0"],
                   "geneo_vectors": info["ngeneo"], "iterations": it, "tol": TOL, "gamma": w.gamma,
                   "variant": args.variant, "parallelism": f"sharded x{world} (setup replicated)",
                   "l2": "flushed between steps (256 MB write)"},
        "iterations": it, "setup_s": setup_s,
        "shard_rank0": {k: v for k, v in sh.items()},
        "roofline": {"bound": "hbm", "kernel": "whole PCG iteration (all ranks)", "achieved": gbs,
                     "peak": peak * world, "unit": "GB/s", "frac": gbs / (peak * world), "traffic": None,
                     "peak_source": src + f" x {world} GPUs", "bytes_per_iteration": bm["iteration"]},
        "e2e": {"value": n * it / (e2e_ms_max / 1e3), "unit": UNIT, "h2d_bytes_per_step": 8 * n_own,
                "d2h_bytes_per_step": 8 * n_own},
        "gpu_launches": int(G.last_launches()) * args.steps,
        "clocks": clocks,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    G.close()


def roofline(G, sweep_ms, in_step, csweep_ms=None, cin_step=(0.0, 0), total_ms=None, cfg=None):
    """Dominant kernel of the step against the measured HBM copy bandwidth
    (MEASURED_PEAKS.json): of the two persistent supernodal sweeps (k_sweep) -- the
    local solves M_AS and the coarse solve E^{-1}, one launch each per PCG
    iteration -- the one with the larger share of the step's device time."""
    peak, src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        pass
    info = G.info
    b = G.bytes_model()["local"]
    achieved = b / (sweep_ms / 1e3) / 1e9
    # the coarse sweep: every factor entry of E once per direction + the right-hand
    # side and solution in coarse positions
    cb = 2 * 8 * info["coarse_factor_nnz"] + 16 * info["n0"]
    coarse = None
    if csweep_ms:
        c_in = cb / (cin_step[0] / 1e3) / 1e9 if cin_step[0] > 0 else None
        coarse = {"kernel": "k_sweep (coarse solve E^-1)", "bytes_per_launch": cb, "avg_launch_ms": csweep_ms,
                  "achieved": cb / (csweep_ms / 1e3) / 1e9, "avg_launch_ms_in_step": cin_step[0],
                  "achieved_in_step": c_in, "launches_in_step": cin_step[1]}
    achieved_in_step = b / (in_step[0] / 1e3) / 1e9 if in_step[0] > 0 else None
    traffic = {}
    try:  # DRAM bytes per launch of both sweeps from the committed ncu --set full capture
        # (tools/gpu_profile_round.sh: tools/ncu_c4.py sweeps launches the local sweep, then E^-1)
        with open(os.path.join(ROOT, "profiles", "r02_ncu_sweeps_c4.json")) as fh:
            cap = json.load(fh)
        if cfg == "c4" and len(cap) == 2:
            traffic = {"local": float(cap[0]["dram_bytes_per_launch"]),
                       "coarse": float(cap[1]["dram_bytes_per_launch"])}
    except Exception:
        pass
    local = {"kernel": "k_sweep (local solves: gather, L y = b, D^-1, L^T x = z, prolong)",
             "achieved": achieved, "bytes_per_launch": b,
             "avg_launch_ms": sweep_ms, "avg_launch_ms_in_step": in_step[0],
             "achieved_in_step": achieved_in_step, "launches_in_step": in_step[1]}
    # dominant = the larger in-step total time (launches x in-kernel duration)
    tl = in_step[0] * in_step[1]
    tc = cin_step[0] * cin_step[1] if coarse else 0.0
    main, other = (coarse, local) if coarse and tc > tl else (local, coarse)
    for k in (main, other):
        if k:
            k["frac"] = k["achieved"] / peak
            k["frac_in_step"] = k["achieved_in_step"] / peak if k["achieved_in_step"] else None
            if total_ms:   # in-kernel time of all its launches / the timed region's device time
                k["share_of_step"] = k["avg_launch_ms_in_step"] * k["launches_in_step"] / total_ms
    if local is not None:
        local["traffic"] = traffic.get("local")
    if coarse is not None:
        coarse["traffic"] = traffic.get("coarse")
    out = {"bound": "hbm", "kernel": main["kernel"], "achieved": main["achieved"], "peak": peak, "unit": "GB/s",
           "frac": main["achieved"] / peak, "traffic": main.get("traffic"),
           "traffic_source": "profiles/r02_ncu_sweeps_c4.json (dram__bytes_read.sum + dram__bytes_write.sum, "
                             "one ncu --set full launch)" if main.get("traffic") else None,
           "peak_source": src,
           "bytes_per_launch": main["bytes_per_launch"], "avg_launch_ms": main["avg_launch_ms"],
           "avg_launch_ms_in_step": main["avg_launch_ms_in_step"], "achieved_in_step": main["achieved_in_step"],
           "frac_in_step": main["frac_in_step"], "launches_in_step": main["launches_in_step"],
           "other_sweep": other}
    return out


if __name__ == "__main__":
    main()
