"""Summarise ncu outputs (gpurun_out/) into profiles/ (committed evidence).

launch list (--metrics gpu__time_duration.sum, cold-cache, serialised) ->
per-kernel-class share; full capture (--set full) -> per-launch DRAM bytes,
throughput, occupancy, registers; writes profiles/ncu_traffic.json
(dram read+write bytes per launch by librk kernel class, for bench.py)."""
import csv
import json
import re
import subprocess
import sys
from collections import defaultdict

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
workload = sys.argv[3] if len(sys.argv) > 3 else "c3"
cmd = sys.argv[4] if len(sys.argv) > 4 else ("python bench.py --steps 1 --warmup 3 --no-cpu-baseline "
                                             "--no-e2e --no-secondary")


def cls_of(name, grid=None):
    m = re.search(r"stencil_kernel<(\d+), (\d+), (\d+)>", name)
    if m:
        mode = int(m.group(2))
        return {0: "stencil_spmv", 1: "stencil_spmv_sweep1", 2: "stencil_sweep", 3: "stencil_sweep",
                4: "stencil_resid", 5: "stencil_resid_sweep1", 6: "stencil_scale"}[mode]
    if "chain19_kernel" in name:
        return "chain19"
    m = re.search(r"chain_kernel(_x2)?<(\d+), (\d+)", name)
    if m:
        return "chain"
    if "rotate_cb_kernel" in name:
        return "rotate"
    for k in ("bdot2", "bupd_gram", "bproj_s", "bdot", "bupd", "normalize", "lincomb", "proj", "rotate", "bicg_p", "bicg_s",
              "bicg_xr", "bicg_setup", "validate", "chain", "invdiag", "colour_sweep"):
        if re.search(rf"\b{k}_(tile_|bulk_)?kernel\b", name):
            return k
        if re.search(rf"\b{k}(_kernel)?\b", name) or f"{k}_kernel" in name:
            return k
    return name.split("(")[0][:40]


rows = list(csv.reader(open(f"{src}/launches.csv")))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[hi + 1:]:
    if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    c = cls_of(r[ki])
    agg[c][0] += 1
    agg[c][1] += v
    tot += v
out = [f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none), "
       f"{sum(a[0] for a in agg.values())} launches of `{cmd}` ({workload} workload; cold-cache, "
       f"serialised => compare SHARES)",
       f"{'class':24s} {'launches':>9s} {'total_us':>12s} {'share':>7s} {'us/launch':>10s}"]
for c, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    out.append(f"{c:24s} {n:9d} {t / 1e3:12.1f} {t / tot:7.3f} {t / 1e3 / n:10.2f}")
open(f"profiles/{tag}_launch_shares.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))

raw = subprocess.run(["ncu", "-i", f"{src}/prof.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h, units = rr[0], rr[1]
want = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
        "smsp__inst_executed.sum"]
idx = {w: h.index(w) for w in want if w in h}


def num(r, w, scale_to):
    i = idx[w]
    v = float(r[i].replace(",", ""))
    u = units[i]
    f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
         "msecond": 1e-3, "second": 1.0, "%": 1, "": 1}.get(u, 1)
    return v * f / scale_to


lines = [f"# {tag}: ncu --set full --clock-control none, selected launches of the same command",
         f"{'kernel':46s} {'grid':>6s} {'regs':>5s} {'us':>8s} {'DRAM MB':>9s} {'GB/s':>7s} {'dram%':>6s} {'warps%':>7s}"]
traffic = defaultdict(list)
for r in rr[2:]:
    name = r[idx["Kernel Name"]]
    t = num(r, "gpu__time_duration.sum", 1.0)
    db = num(r, "dram__bytes_read.sum", 1.0) + num(r, "dram__bytes_write.sum", 1.0)
    c = cls_of(name)
    traffic[c].append(db)
    lines.append(f"{name.split('(')[0][-46:]:46s} {r[idx['launch__grid_size']]:>6s} "
                 f"{r[idx['launch__registers_per_thread']]:>5s} {t * 1e6:8.1f} {db / 1e6:9.1f} "
                 f"{db / t / 1e9:7.0f} {float(r[idx['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']]):6.1f} "
                 f"{float(r[idx['sm__warps_active.avg.pct_of_peak_sustained_active']]):7.1f}")
open(f"profiles/{tag}_ncu_full_summary.txt", "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
tj = {c: sum(v) / len(v) for c, v in traffic.items()}
try:
    old = json.load(open("profiles/ncu_traffic.json"))
except (OSError, ValueError):
    old = {}
old = {k: v for k, v in old.items() if isinstance(v, dict)}
old[workload] = {"_note": f"{tag}: mean dram__bytes_read.sum + dram__bytes_write.sum per launch "
                          "(bytes) from the ncu --set full capture; keyed by librk kernel class",
                 **{k: round(v) for k, v in tj.items()}}
json.dump(old, open("profiles/ncu_traffic.json", "w"), indent=1)
