"""Build librk with extra -D flags into scripts/micro/<name>/librk.so (experiments)."""
import os, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_1501_03358_b200 import build as B
name, defs = sys.argv[1], sys.argv[2:]
out = os.path.join(ROOT, "scripts", "micro", name)
os.makedirs(out, exist_ok=True)
jobs = [(B.flags(defs) + ["-c", os.path.join(B.CSRC, s), "-o", os.path.join(out, s + ".o")]) for s in B.SOURCES]
with ThreadPoolExecutor(len(jobs)) as ex:
    for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs):
        if r.returncode:
            sys.exit(r.stderr[-3000:])
link = [B.nvcc_path(), *B.ARCH, "-shared", *[j[-1] for j in jobs], "-o", os.path.join(out, "librk.so"), "-lcudart"]
if B.have_nccl():
    link.append("-lnccl")
subprocess.run(link, check=True)
print(os.path.join(out, "librk.so"))
