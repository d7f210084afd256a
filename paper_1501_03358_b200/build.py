"""Build librk.so in-tree with nvcc for sm_100a (no JIT, no torch extension
machinery).  Used by __graft_entry__.build() and `python -m
paper_1501_03358_b200.build`."""
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "librk.so")
SOURCES = ["stencil.cu", "blockops.cu", "bicg.cu", "chain.cu", "librk.cpp", "comm.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def have_nccl():
    return os.path.exists("/usr/include/nccl.h")


def flags(extra=()):
    f = [nvcc_path(), "-std=c++17", "-O3", "-lineinfo", *ARCH, "-Xcompiler", "-fPIC",
         "-Xcompiler", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
         "-Xptxas", "-warn-spills"]
    if have_nccl():
        f += ["-DRK_WITH_NCCL"]
    return f + list(extra)


def command(out=LIB, extra=()):
    """Single-invocation build command (documentation / manual builds)."""
    cmd = flags(extra) + ["-shared"] + [os.path.join(CSRC, s) for s in SOURCES]
    cmd += ["-o", out, "-lcudart"]
    if have_nccl():
        cmd += ["-lnccl"]
    return cmd


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "rk.h"))
    deps.append(os.path.abspath(__file__))
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force=False, verbose=True):
    if not force and up_to_date():
        return LIB
    # one nvcc per translation unit, in parallel, then one link
    from concurrent.futures import ThreadPoolExecutor
    odir = os.path.join(HERE, "build_obj")
    os.makedirs(odir, exist_ok=True)
    objs = [os.path.join(odir, s + ".o") for s in SOURCES]
    cmds = [flags() + ["-c", os.path.join(CSRC, s), "-o", o] for s, o in zip(SOURCES, objs)]
    if verbose:
        for c in cmds:
            print(" ".join(c), flush=True)
    with ThreadPoolExecutor(len(cmds)) as ex:
        for r in ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds):
            sys.stdout.write(r.stdout)
            sys.stderr.write(r.stderr)
            if r.returncode != 0:
                raise subprocess.CalledProcessError(r.returncode, r.args)
    tmp = LIB + ".tmp"
    link = [nvcc_path(), *ARCH, "-shared", *objs, "-o", tmp, "-lcudart"]
    if have_nccl():
        link += ["-lnccl"]
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
