"""Build an A/B variant of librk with extra compile-time defines for chain.cu
(e.g. -DRK_C19_ROT=0) into paper_1501_03358_b200/variants/librk_<tag>.so;
bench.py / tests load it when RK_LIBPATH points at it (measurement only --
the product path is the in-tree librk.so).
usage: python scripts/build_variant.py <tag> [--src=file.cu] -DNAME=VALUE ...
(--src: the translation unit the defines apply to; default chain.cu)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1501_03358_b200 import build as B  # noqa: E402

tag, defs = sys.argv[1], sys.argv[2:]
src = "chain.cu"
for a in list(defs):
    if a.startswith("--src="):
        src = a.split("=", 1)[1]
        defs.remove(a)
B.build(verbose=False)
odir = os.path.join(B.HERE, "build_obj")
vdir = os.path.join(B.HERE, "variants")
os.makedirs(vdir, exist_ok=True)
vobj = os.path.join(vdir, f"{src}_{tag}.o")
subprocess.run(B.flags(defs) + ["-c", os.path.join(B.CSRC, src), "-o", vobj], check=True)
objs = [vobj if s == src else os.path.join(odir, s + ".o") for s in B.SOURCES]
out = os.path.join(vdir, f"librk_{tag}.so")
link = [B.nvcc_path(), *B.ARCH, "-shared", *objs, "-o", out, "-lcudart"]
if B.have_nccl():
    link += ["-lnccl"]
subprocess.run(link, check=True)
print(out)
