#!/usr/bin/env python
"""Benchmark of the recycling-Krylov hot path on B200.

A "step" is one pass of the whole hot path (every SURVEY §8(a) row) over
one batch of synthetic input: the full 20-system hybrid sequence of
BASELINE configs[2] (128^3 porous 7-point operator; rGCROT(10,20) with
p1 = 2 for systems 0-2, then rBiCGStab recycling the frozen space), solved
from an empty recycle space.  configs[2] is the BASELINE config that runs
every §8(a) row (configs[1] never reaches rBiCGStab) and fits one GPU.

metric: BASELINE.json's; value = solve ms per system (lower is better),
whole job.  With torchrun (N > 1) every rank owns a z-slab of the same grid
(strong scaling; NCCL halo + allreduce inside librk).

`--impl reference` times the CPU oracle (this tier's reference arm) on a
bounded sample of the same workload.
"""
import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "solve ms/system & iterations; SpMV+projection HBM GB/s vs roofline, 1–8 B200"
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="rk", choices=["rk", "reference"])
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-sample-seconds", type=float, default=20.0)
    ap.add_argument("--breakdown", action="store_true", help="print per-kernel-class shares")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return FALLBACK_HBM, "fallback"


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
def cpu_sample(workload, seconds, gpu_mv=None):
    """The oracle as it stands, timed on this host on a bounded sample of
    the workload: (a) one rGCROT(m, k) cycle of system 0 (m Krylov matvecs),
    (b) rBiCGStab iterations of system n_sw with a k-dim recycle space
    (random U refreshed by QR -- iteration cost does not depend on the
    space's quality).  Extrapolated to ms/system with the per-system Krylov
    matvec counts of the GPU run (same algorithm; parity within 10 %)."""
    from dataclasses import replace
    from oracle.krylov import rbicgstab, refresh_space, rgcrot
    from oracle.stencil import Jacobi, Operator
    from problems import get_workload
    w = get_workload(workload)
    prm = w.params
    prob = w.problem()
    t0 = time.perf_counter()
    op = Operator.from_problem(prob)
    pc = Jacobi(op, prm.sweeps, prm.omega_l, prm.omega_g)
    setup = time.perf_counter() - t0
    b0 = prob.rhs(0).reshape(-1)
    e = np.zeros((prob.N, 0))
    t0 = time.perf_counter()
    _, _, _, r1 = rgcrot(op, pc, b0, e, e, replace(prm, max_mv=prm.m, tol=1e-30))
    t_rg = time.perf_counter() - t0
    ms_rg = 1e3 * t_rg / max(1, r1.krylov_mv)
    ms_bi = None
    if prm.method == "hybrid":
        U0 = np.random.default_rng(0).uniform(-1, 1, (prob.N, prm.k_max))
        U, C, _ = refresh_space(op.apply, U0)
        budget = max(4, int(2 * max(1.0, seconds - t_rg) / max(1e-3, 2 * ms_rg / 1e3)) // 2 * 2)
        budget = min(budget, 20)
        t0 = time.perf_counter()
        _, _, _, r2 = rbicgstab(op, pc, prob.rhs(prm.n_sw).reshape(-1), U, C,
                                replace(prm, max_mv=budget, tol=1e-30), valid=True)
        t_bi = time.perf_counter() - t0
        ms_bi = 1e3 * t_bi / max(1, r2.krylov_mv)
    sample = (f"{workload}: oracle rGCROT cycle of system 0 ({r1.krylov_mv} Krylov matvecs, "
              f"{ms_rg:.0f} ms/matvec)")
    if ms_bi is not None:
        sample += f" + rBiCGStab k={prm.k_max} ({r2.krylov_mv} matvecs, {ms_bi:.0f} ms/matvec)"
    est = None
    if gpu_mv is not None:
        tot = 0.0
        for tag, mv in gpu_mv:
            tot += mv * (ms_bi if (tag == "rbicgstab" and ms_bi) else ms_rg)
        est = tot / len(gpu_mv)
        sample += "; extrapolated to ms/system with the GPU run's per-system matvec counts"
    return {"ms_per_mv_rgcrot": ms_rg, "ms_per_mv_rbicgstab": ms_bi, "ms_per_system": est,
            "sample": sample, "setup_s": setup}


def oracle_counts(workload):
    """[(tag, krylov matvecs)] of the oracle's full sequence, if stored."""
    p = os.path.join(ROOT, "tests", "golden", f"oracle_seq_{workload}.json")
    if not os.path.exists(p):
        return None, None
    d = json.load(open(p))
    return ([[r["tag"], r["krylov_matvecs"]] for r in d["systems"]],
            f"the oracle's own full-sequence counts ({os.path.relpath(p, ROOT)})")


def run_reference(args):
    """--impl reference: the CPU oracle, timed per step on a bounded sample."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from problems import get_workload
    w = get_workload(args.workload)
    # each step times one rGCROT cycle + rBiCGStab iterations of the oracle
    ms = []
    info = None
    for i in range(args.warmup + args.steps):
        info = cpu_sample(args.workload, max(2.0, args.cpu_sample_seconds / 4))
        if i >= args.warmup:
            ms.append(info)
    mrg = float(np.mean([m["ms_per_mv_rgcrot"] for m in ms]))
    mbi = [m["ms_per_mv_rbicgstab"] for m in ms if m["ms_per_mv_rbicgstab"]]
    mbi = float(np.mean(mbi)) if mbi else mrg
    # ms/system for the sequence with the oracle's OWN per-system Krylov
    # matvec counts (tests/golden/oracle_seq_<workload>.json, written by
    # scripts/oracle_counts.py from oracle/ alone); without that file, the
    # hybrid's structure at 100 matvecs per system.
    counts, src = oracle_counts(args.workload)
    if not counts:
        counts = [["rgcrot" if t < w.params.n_sw else "rbicgstab", 100] for t in range(w.n_systems)]
        src = "100 matvecs/system assumed"
    value = sum(mv * (mbi if tag == "rbicgstab" else mrg) for tag, mv in counts) / len(counts)
    cores = os.cpu_count()
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "ms/system",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(value * len(counts), 3), "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.description}",
                   "systems": w.n_systems, "l2": "inputs larger than L2"},
        "cpu_baseline": {"value": round(value, 3), "unit": "ms/system", "cores": cores,
                         "kind": "oracle", "sample": ms[-1]["sample"] +
                         f"; per-system matvecs: {src}"
                         " (NumPy; stencil and elementwise work single-threaded)"},
        "e2e": {"value": round(value, 3), "unit": "ms/system", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    z0, z1 = slab_range(prob.nz, rank, world)
    uid = None
    if world > 1:
        obj = [rk.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = rk.Context(local, rank, world, uid)
    stream = torch.cuda.current_stream()
    bands = torch.from_numpy(prob.bands(z0, z1, epoch=w.epoch(0))).cuda()
    op = rk.GridOperator(ctx, prob.nx, prob.ny, prob.nz, prob.offsets, bands, prob.periodic,
                         z0=z0, nz_local=z1 - z0)
    del bands
    solver = rk.Solver(op, rk.config_from_params(prm))
    T = w.n_systems
    Nl = op.N
    B = [torch.from_numpy(prob.rhs(t, z0, z1).reshape(-1)).cuda() for t in range(T)]
    X = [torch.zeros(Nl, dtype=torch.float64, device="cuda") for _ in range(T)]
    epoch_bands = {}

    def bands_for(e):
        if e not in epoch_bands:
            epoch_bands[e] = torch.from_numpy(prob.bands(z0, z1, epoch=e)).cuda()
        return epoch_bands[e]

    def step(host=False, Bh=None, Xh=None):
        solver.recycle_set(None)                      # fresh, empty recycle space
        if w.epoch_every and w.epoch(0) != w.epoch(T - 1):
            op.update_bands(bands_for(w.epoch(0)))
        return rk.solve_sequence(solver, (lambda t: Bh[t]) if host else (lambda t: B[t]), T,
                                 prm.method, n_sw=prm.n_sw, epoch_of=w.epoch,
                                 bands_for_epoch=bands_for, host=host,
                                 x_out=Xh if host else X)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, args.warmup)):
        reps = step()
    # kernel-class breakdown (untimed pass, every launch bracketed by events)
    ctx.profile(True, None)
    ctx.profile_read(reset=True)
    step()
    prof_all = ctx.profile_read()
    ctx.profile(False)
    ctx.profile_read(reset=True)
    dominant = max(prof_all.items(), key=lambda kv: kv[1]["ms"])[0]
    # timed region
    clocks = Clocks(local) if rank == 0 else None
    # live timing of the dominant class inside the timed region: every 8th
    # launch is bracketed by events (fewer event records in the timed loop)
    ctx.profile(True, dominant, every=8)
    launches0 = ctx.launches()
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    all_reps = []
    for _ in range(args.steps):
        all_reps.append(step())
    ev1.record(stream)
    barrier()
    ms = ev0.elapsed_time(ev1)
    launches = ctx.launches() - launches0
    prof_dom = ctx.profile_read().get(dominant, {"launches": 0, "ms": 0.0, "bytes": 0.0})
    ctx.profile(False)
    ctx.profile_read(reset=True)
    clk = clocks.stop() if clocks else None
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    reps = all_reps[-1]
    ms_per_step = ms / args.steps
    value = ms_per_step / T
    mv = [r["krylov_matvecs"] for r in reps]
    # e2e: host buffers through rk_solve_host, copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Bh = [b.cpu().pin_memory() for b in B]
        Xh = [torch.zeros(Nl, dtype=torch.float64).pin_memory() for _ in range(T)]
        step(True, Bh, Xh)
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(True, Bh, Xh)
        e1.record(stream)
        barrier()
        wall = e0.elapsed_time(e1)   # device time on the library stream; copies included
        if world > 1:
            t = torch.tensor([wall], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            wall = float(t.item())
        e2e = {"value": round(wall / args.steps / T, 3), "unit": "ms/system",
               "h2d_bytes_per_step": int(T * Nl * 8 * world),      # b_t (x0 = 0 is not uploaded)
               "d2h_bytes_per_step": int(T * Nl * 8 * world)}
    if rank != 0:
        return
    peak, peak_kind = peaks()
    achieved = prof_dom["bytes"] / (prof_dom["ms"] * 1e-3) / 1e9 if prof_dom["ms"] > 0 else None
    traffic = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(dominant)
    total_ms = sum(v["ms"] for v in prof_all.values())
    # whole-step effective bandwidth of the algorithmic bytes of every kernel
    alg_bytes = sum(v["bytes"] for v in prof_all.values())
    line = {
        "metric": METRIC, "value": round(value, 4), "unit": "ms/system", "n_gpus": world,
        "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w.description}", "grid": [prob.nx, prob.ny, prob.nz],
                   "systems": T, "method": prm.method, "m": prm.m, "k": prm.k_max, "p1": prm.p1,
                   "n_sw": prm.n_sw, "tol": prm.tol, "parallelism": f"z-slab x{world}",
                   "l2": "inputs larger than L2 (bases+bands ~ 1 GB at 128^3)"},
        "iterations": {"krylov_matvecs_per_system": mv, "mean": float(np.mean(mv)),
                       "outcomes": sorted(set(r["outcome"] for r in reps)),
                       "tags": [r["tag"] for r in reps]},
        "roofline": {"bound": "hbm", "kernel": dominant,
                     "achieved": round(achieved, 1) if achieved else None, "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4) if achieved else None,
                     "peak_kind": peak_kind, "traffic": traffic,
                     "frac_of_8TBs": round(achieved / 8000.0, 4) if achieved else None,
                     "launches_timed": prof_dom["launches"], "timed_every": 8,
                     "share_of_step": round(prof_all[dominant]["ms"] / total_ms, 4) if total_ms else None},
        "step_effective_gbs": round(alg_bytes / (total_ms * 1e-3) / 1e9, 1) if total_ms else None,
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
    }
    if True:   # per-kernel-class breakdown of the untimed profiling pass
        line["kernel_breakdown"] = {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                                        "gbs": round(v["bytes"] / (v["ms"] * 1e-3) / 1e9, 1) if v["ms"] else None}
                                    for k, v in sorted(prof_all.items(), key=lambda kv: -kv[1]["ms"])}
    if world == 1 and not args.no_cpu_baseline:
        counts, src = oracle_counts(args.workload)
        if not counts:
            counts, src = [(r["tag"], r["krylov_matvecs"]) for r in reps], "the GPU run's per-system counts"
        cb = cpu_sample(args.workload, args.cpu_sample_seconds, counts)
        cb["sample"] = cb["sample"].replace("the GPU run's per-system matvec counts", src)
        line["cpu_baseline"] = {"value": round(cb["ms_per_system"], 1), "unit": "ms/system",
                                "cores": os.cpu_count(), "kind": "oracle", "sample": cb["sample"]}
    print(json.dumps(line), flush=True)
    solver.close()
    op.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_rk(args)


if __name__ == "__main__":
    main()
