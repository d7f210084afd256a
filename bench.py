#!/usr/bin/env python
"""Benchmark of the recycling-Krylov hot path on B200.

Workload (default): BASELINE configs[3], the largest configuration that
fits one GPU -- the 256^3 19-point channel-shaped operator (periodic x/z,
Neumann y, one pinned dof), a 50-system sequence b_t = b_0 + 0.05 t
noise_t with A perturbed by 1e-3 relative every 10 systems, solved by
rGCROT(40,30) (p1 = 1, Jacobi(5+1)), carrying the recycle space from
system to system (PAPER P:687-704 is the paper's channel case).

A "step" is one system of that sequence, in order: warm-up steps solve
systems 0 .. W-1 (untimed; they grow the recycle space from empty), the K
timed steps solve systems W .. W+K-1, including every A-epoch change
(bands upload + recycle-space refresh) that falls in that range; the
sequence is cyclic past its 50th system.  metric: BASELINE.json's; value
= device ms per system over the K timed systems (lower is better).  With
torchrun (N > 1) every rank owns a z-slab of the same grid (strong
scaling; NCCL halo + allreduce inside librk).

`e2e` replays the same K systems from the same recycle-space state
(exported after the warm-up, re-imported through rk_recycle_set) through
the pipelined host-buffer API: every b_t upload and x_t download is
inside the timed region.  `secondary` is BASELINE configs[2] (128^3 porous
hybrid, one step = the whole 20-system sequence from an empty space).

`--impl reference` times the CPU oracle (this tier's reference arm) on a
bounded sample of the same workload.
"""
import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve ms/system & iterations; SpMV+projection HBM GB/s vs roofline, 1–8 B200"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="rk", choices=["rk", "reference"])
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--secondary", default="c3")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        time.sleep(0.25)
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [ln.split(",") for ln in open(self.f.name).read().splitlines() if ln.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                for nm, v in zip(names, r[5:9]):
                    if v.strip() == "Active":
                        reasons.add(nm)
            except (ValueError, IndexError):
                pass
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ oracle
def oracle_matvec_sample(workload, planes=32, threads=None):
    """The oracle as it stands (oracle.krylov.rgcrot, untuned), timed on this
    host on a bounded sample: the workload's operator on its first `planes`
    z-planes (a grid of its own; every oracle operation is linear in N, so
    times scale by nz / planes -- checked: 32 and 64 planes of c4 take 7.7 and
    15.0 s per m = 1 cycle), a recycle space of k + m/2 columns (the average
    [C V_j] width of an rGCROT(m, k) cycle; a random orthonormal C -- the cost
    does not depend on the space's quality) and one rGCROT cycle with m = 1
    and one with m = 4 Krylov steps.  A third of their difference is the
    marginal cost of a Krylov matvec (the preconditioned operator application
    and its CGS2 orthogonalisation); the rest of the m = 1 cycle is the
    per-cycle cost (the
    M^-1 b / re-projection at the start, the cycle end's update, true
    residual and line-14a update).  Returns full-grid ms per Krylov matvec,
    ms per cycle, and the space width."""
    from dataclasses import replace
    from oracle.krylov import rgcrot
    from oracle.stencil import Jacobi, Operator
    from problems import get_workload
    w = get_workload(workload)
    prm = w.params
    prob = w.problem()
    nz = min(planes, prob.nz)
    op = Operator(prob.nx, prob.ny, nz, prob.periodic, prob.offsets, prob.bands(0, nz), check=False)
    pc = Jacobi(op, prm.sweeps, prm.omega_l, prm.omega_g)
    b = prob.rhs(0, 0, nz).reshape(-1)
    kk = prm.k_max + prm.m // 2
    rng = np.random.default_rng(0)
    C, _ = np.linalg.qr(rng.standard_normal((op.N, kk)))
    U = rng.standard_normal((op.N, kk))

    def cycle(m):
        t0 = time.perf_counter()
        _, _, _, rep = rgcrot(op, pc, b, U, C, replace(prm, m=m, k_max=kk + 2, max_mv=m, tol=1e-30),
                              valid=True)
        assert rep.krylov_mv == m and rep.cycles == 1
        return time.perf_counter() - t0

    def both():
        return cycle(1), cycle(4)

    if threads is None:
        t1, t2 = both()
    else:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=threads):
            t1, t2 = both()
    scale = 1e3 * prob.nz / nz
    mv = max(t2 - t1, 0.0) / 3.0
    return mv * scale, max(t1 - mv, 0.0) * scale, kk, nz


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """--impl reference: the CPU oracle, one bounded sample per step (the
    two cycles of oracle_matvec_sample on the first 8 z-planes,
    scaled to the full grid), composed into ms per system with the
    workload's Krylov matvecs and cycles per system (below)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from problems import get_workload
    w = get_workload(args.workload)
    mvs, cys = [], []
    kk = nz = None
    walls = []
    for i in range(args.warmup + args.steps):   # 8 planes: ~6 s per step on the box's host (default 25 steps: ~3 min)
        t0 = time.perf_counter()
        a, c, kk, nz = oracle_matvec_sample(args.workload, planes=8)
        if i >= args.warmup:
            mvs.append(a)
            cys.append(c)
            walls.append((time.perf_counter() - t0) * 1e3)
    ms_mv, ms_cy = float(np.mean(mvs)), float(np.mean(cys))
    mv_sys = MV_PER_SYSTEM.get(args.workload, 100.0)
    cy_sys = mv_sys / w.params.m
    value = ms_mv * mv_sys + ms_cy * cy_sys
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms/system",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # a step is one bounded sample (wall time as run); value is the
        # sample's ms per matvec / per cycle composed into ms per system
        "ms_per_step": round(float(np.mean(walls)), 3), "value_is": "extrapolated from the per-step samples",
        "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.description}", "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/system", "cores": cores,
                         "cpu_model": cpu_model(), "kind": "oracle",
                         "sample": (f"per step: oracle rGCROT cycles with m=1 and m=4 Krylov steps against "
                                    f"a {kk}-column recycle space on the first {nz} z-planes of the "
                                    f"{args.workload} grid, scaled to the full grid: {ms_mv:.0f} ms per "
                                    f"Krylov matvec + {ms_cy:.0f} ms per cycle, x {mv_sys} matvecs and "
                                    f"{cy_sys:.1f} cycles per system ({MV_SOURCE}) (NumPy; stencil and "
                                    f"elementwise work single-threaded, BLAS on all cores)")},
        "e2e": {"value": round(value, 3), "unit": "ms/system", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# Krylov matvecs per system used to turn the oracle's ms per matvec into ms
# per system in the reference arm (a separate process that cannot see the
# GPU arm's counts): the mean over systems 5-24 of the c4 rGCROT(40,30) T2
# run (profiles/r02_bench_c4_nfuse.json); GPU and oracle counts agree per system
# within one cycle (tests/gpu/test_gpu_parity.py).  The GPU arm's own
# cpu_baseline uses the counts of its own timed systems.
MV_PER_SYSTEM = {"c4": 438.0, "c3": 179.5}
MV_SOURCE = "mean Krylov matvecs per timed system of the GPU run, profiles/r02_bench_c4_nfuse.json"


# ------------------------------------------------------------------ GPU arm
def run_rk(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1501_03358_b200 as rk
    from problems import get_workload, slab_range

    w = get_workload(args.workload)
    prm = w.params
    prob = w.problem()
    T = w.n_systems
    W = max(3, args.warmup)
    K = args.steps
    z0, z1 = slab_range(prob.nz, rank, world)
    uid = None
    if world > 1:
        obj = [rk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = rk.Context(local, rank, world, uid)
    stream = torch.cuda.current_stream()
    epoch_of = lambda s: w.epoch(s % T)          # cyclic sequence
    epoch_bands = {epoch_of(0): torch.from_numpy(prob.bands(z0, z1, epoch=epoch_of(0))).cuda()}

    def bands_for(e):
        if e not in epoch_bands:
            epoch_bands[e] = torch.from_numpy(prob.bands(z0, z1, epoch=e)).cuda()
        return epoch_bands[e]

    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, bands_for(epoch_of(0)),
                         prob.periodic, z0=z0, nz_local=z1 - z0)
    solver = rk.Solver(op, rk.config_from_params(prm))
    Nl = op.N
    # right-hand sides of every system the run touches, resident in HBM
    ts = sorted({s % T for s in range(W + K)})
    with ThreadPoolExecutor(8) as ex:
        host_b = dict(zip(ts, ex.map(lambda t: prob.rhs(t, z0, z1).reshape(-1), ts)))
    B = {t: torch.from_numpy(host_b[t]).cuda() for t in ts}
    for s in range(W + K):                     # every epoch's bands before timing
        bands_for(epoch_of(s))
    X = torch.zeros(Nl, dtype=torch.float64, device="cuda")

    def solve(s0, n, host=False, Bh=None, Xh=None):
        return rk.solve_sequence(solver, (lambda s: Bh[s % T]) if host else (lambda s: B[s % T]), n,
                                 prm.method, n_sw=prm.n_sw, epoch_of=epoch_of,
                                 bands_for_epoch=bands_for, host=host,
                                 x_out=Xh[s0:s0 + n] if host else [X] * n, start=s0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up: systems 0 .. W-2 plain, system W-1 with every launch bracketed
    # (kernel-class breakdown; the arithmetic is unchanged)
    solver.recycle_set(None)
    wreps = solve(0, W - 1)
    ctx.profile(True, None)
    ctx.profile_read(reset=True)
    wreps += solve(W - 1, 1)
    prof_all = ctx.profile_read()
    ctx.profile(False)
    ctx.profile_read(reset=True)
    dominant = max(prof_all.items(), key=lambda kv: kv[1]["ms"])[0]
    # recycle-space state entering the timed region (for the e2e replay)
    U0, C0, _ = solver.recycle_export()
    # timed region: systems W .. W+K-1; live event timing of every 8th
    # launch of the dominant kernel class
    clocks = Clocks(local) if rank == 0 else None
    ctx.profile(True, dominant, every=8)
    launches0 = ctx.launches()
    coll0 = ctx.comm_count()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    reps = solve(W, K)
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - launches0
    coll1 = ctx.comm_count()
    prof_dom = ctx.profile_read().get(dominant, {"launches": 0, "ms": 0.0, "bytes": 0.0})
    ctx.profile(False)
    ctx.profile_read(reset=True)
    clk = clocks.stop() if clocks else None
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ms / K
    mv = [r["krylov_matvecs"] for r in reps]
    cycles = [r["cycles_or_iters"] for r in reps]
    outcomes = [r["outcome"] for r in reps]
    # e2e: the same K systems from the same recycle-space state, host buffers
    e2e = None
    if not args.no_e2e:
        Bh = {t: torch.from_numpy(host_b[t]).pin_memory() for t in ts}
        Xh = [torch.zeros(Nl, dtype=torch.float64).pin_memory() for _ in range(W + K)]
        op.update_bands(bands_for(epoch_of(W - 1)))
        solver.set_method("rgcrot" if prm.method in ("rgcrot", "gmres") or W - 1 < prm.n_sw
                          else "rbicgstab")
        solver.recycle_set(U0, C0)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ereps = solve(W, K, True, Bh, Xh)
        e1.record(stream)
        barrier()
        wall = e0.elapsed_time(e1)   # device time on the library stream; copies included
        if world > 1:
            t = torch.tensor([wall], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        e2e = {"value": round(wall / K, 3), "unit": "ms/system",
               "h2d_bytes_per_step": int(Nl * 8 * world),      # b_t (x0 = 0 is not uploaded)
               "d2h_bytes_per_step": int(Nl * 8 * world),      # x_t
               "same_matvecs_as_device_run": [r["krylov_matvecs"] for r in ereps] == mv}
    del U0, C0
    secondary = None
    if not args.no_secondary and args.secondary and args.secondary != args.workload and world == 1:
        secondary = sequence_bench(rk, ctx, args.secondary)
    if rank != 0:
        return
    peak, peak_kind = peaks()
    achieved = prof_dom["bytes"] / (prof_dom["ms"] * 1e-3) / 1e9 if prof_dom["ms"] > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(args.workload, {}).get(dominant)
    total_ms = sum(v["ms"] for v in prof_all.values())
    alg_bytes = sum(v["bytes"] for v in prof_all.values())
    epochs = sorted({epoch_of(s) for s in range(W, W + K)})
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/system", "n_gpus": world,
        "steps": K, "warmup": W, "ms_per_step": round(value, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.description}", "grid": [prob.nx, prob.ny, prob.nz],
                   "step": "one system of the sequence, in order",
                   "timed_systems": f"{W}..{W + K - 1} (mod {T})", "epochs_in_timed_region": epochs,
                   "method": prm.method, "m": prm.m, "k": prm.k_max, "k_t": prm.k_t, "p1": prm.p1,
                   "tol": prm.tol, "precond": "jacobi(5+1)", "ortho": "cgs2 gram-corrected (R19)",
                   "parallelism": f"z-slab x{world}",
                   "l2": "inputs larger than L2 (bases + bands per rank ~ %.1f GB)"
                         % (8e-9 * Nl * ((prm.m + 1) + 2 * prm.k_max + (2 if prm.p1 == 2 else 0) + 8
                                         + len(prob.offsets) + 1))},
        "iterations": {"krylov_matvecs_per_system": mv, "mean": float(np.mean(mv)),
                       "recycle_dim_after": [r["k_after"] for r in reps],
                       "outcomes": sorted(set(outcomes)),
                       "ms_per_matvec": round(ms / max(1, sum(mv)), 4)},
        "valid": all(o == "CONVERGED" for o in outcomes),
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                     "peak_kind": peak_kind, "traffic": traffic,
                     "frac_of_8TBs": round(achieved / 8000.0, 4) if achieved else None,
                     "launches_timed": prof_dom["launches"], "timed_every": 8,
                     "share_of_step": round(prof_all[dominant]["ms"] / total_ms, 4) if total_ms else None},
        "step_effective_gbs": round(alg_bytes / (total_ms * 1e-3) / 1e9, 1) if total_ms else None,
        "gpu_launches": launches,
        # collective launches per rank inside the timed region (0 on one GPU)
        "collectives": {"allreduce": coll1[0] - coll0[0], "halo": coll1[1] - coll0[1],
                        "allreduce_per_matvec": round((coll1[0] - coll0[0]) / max(1, sum(mv)), 3),
                        "halo_per_matvec": round((coll1[1] - coll0[1]) / max(1, sum(mv)), 3)},
        "clocks": clk,
        "e2e": e2e,
        "kernel_breakdown": {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                                 "gbs": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                             for k, v in sorted(prof_all.items(), key=lambda kv: -kv[1]["ms"])},
    }
    if not line["valid"]:
        line["invalid_reason"] = "a timed system did not converge: " + ",".join(outcomes)
    if secondary:
        line["secondary"] = secondary
    solver.close()
    op.close()
    epoch_bands.clear()
    B.clear()
    torch.cuda.empty_cache()
    if world == 1 and not args.no_cpu_baseline:
        a_all, c_all, kk, nzs = oracle_matvec_sample(args.workload)
        a_one, c_one, _, _ = oracle_matvec_sample(args.workload, threads=1)
        mvs = float(np.mean(mv))
        cys = float(np.mean(cycles))
        line["cpu_baseline"] = {
            "value": round(a_all * mvs + c_all * cys, 1), "unit": "ms/system", "cores": os.cpu_count(),
            "value_1thread": round(a_one * mvs + c_one * cys, 1), "cpu_model": cpu_model(), "kind": "oracle",
            "sample": (f"oracle rGCROT cycles with m=1 and m=4 Krylov steps against a {kk}-column recycle "
                       f"space (the average [C V_j] width of an rGCROT({prm.m},{prm.k_max}) cycle) on the "
                       f"first {nzs} z-planes of the {prob.nx}x{prob.ny}x{prob.nz} grid, scaled to the full "
                       f"grid: {a_all:.0f} ms per Krylov matvec + {c_all:.0f} ms per cycle with BLAS on all "
                       f"{os.cpu_count()} cores ({a_one:.0f} + {c_one:.0f} ms on 1 thread); times the GPU "
                       f"run's {mvs:.1f} Krylov matvecs and {cys:.1f} cycles per timed system (NumPy "
                       f"stencil and elementwise work is single-threaded in both settings)")}
    text = json.dumps(line)
    print(text, flush=True)
    if args.out:
        open(args.out, "w").write(text + "\n")
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def sequence_bench(rk, ctx, name, steps=3, warmup=2):
    """A whole sequence per step, from an empty recycle space (r01's c3
    measurement): device-resident and through the pipelined host API."""
    import torch
    from problems import get_workload
    w = get_workload(name)
    prm = w.params
    prob = w.problem()
    T = w.n_systems
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets,
                         torch.from_numpy(prob.bands(epoch=w.epoch(0))).cuda(), prob.periodic)
    solver = rk.Solver(op, rk.config_from_params(prm))
    hb = [prob.rhs(t).reshape(-1) for t in range(T)]
    B = [torch.from_numpy(b).cuda() for b in hb]
    X = [torch.zeros(op.N, dtype=torch.float64, device="cuda") for _ in range(T)]
    bands = {}

    def bands_for(e):
        if e not in bands:
            bands[e] = torch.from_numpy(prob.bands(epoch=e)).cuda()
        return bands[e]

    def seq(host=False, Bh=None, Xh=None):
        solver.recycle_set(None)
        if w.epoch_every:
            op.update_bands(bands_for(w.epoch(0)))
        return rk.solve_sequence(solver, (lambda t: Bh[t]) if host else (lambda t: B[t]), T,
                                 prm.method, n_sw=prm.n_sw, epoch_of=w.epoch,
                                 bands_for_epoch=bands_for, host=host, x_out=Xh if host else X)

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        seq()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        reps = seq()
    e1.record(stream)
    torch.cuda.synchronize()
    value = e0.elapsed_time(e1) / steps / T
    Bh = [torch.from_numpy(b).pin_memory() for b in hb]
    Xh = [torch.zeros(op.N, dtype=torch.float64).pin_memory() for _ in range(T)]
    seq(True, Bh, Xh)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(steps):
        seq(True, Bh, Xh)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e = e0.elapsed_time(e1) / steps / T
    mv = [r["krylov_matvecs"] for r in reps]
    solver.close()
    op.close()
    return {"workload": f"{name}: {w.description}", "step": "the whole sequence from an empty space",
            "steps": steps, "warmup": warmup, "value": round(value, 4), "unit": "ms/system",
            "e2e": round(e2e, 4), "matvecs_per_system": mv,
            "outcomes": sorted(set(r["outcome"] for r in reps)),
            "tags": [r["tag"] for r in reps]}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_rk(args)


if __name__ == "__main__":
    main()
