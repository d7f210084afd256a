"""CPU-side checks of the boundary: librk.so builds for sm_100a, loads,
exports every symbol include/rk.h declares, and the ctypes structs match
the header's layout.  No compute calls (there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def librk():
    from paper_1501_03358_b200.build import build
    build()
    from paper_1501_03358_b200 import _lib
    return _lib


def header_functions():
    txt = open(os.path.join(ROOT, "include", "rk.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(rk_[a-z_0-9]+)\s*\(", txt)))


def test_every_declared_symbol_is_exported(librk):
    L = librk.lib()
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(librk.EXPORTED) == declared


def test_nm_shows_extern_c_symbols(librk):
    out = subprocess.run(["nm", "-D", "--defined-only", librk.LIBPATH], capture_output=True,
                         text=True, check=True).stdout
    syms = {line.split()[-1] for line in out.splitlines() if line.strip()}
    for name in header_functions():
        assert name in syms, name


def test_sass_is_sm100a(librk):
    out = subprocess.run(["cuobjdump", "--list-elf", librk.LIBPATH], capture_output=True,
                         text=True, check=True).stdout
    assert "sm_100a" in out


def test_version_and_error_string(librk):
    L = librk.lib()
    assert b"sm_100a" in L.rk_version()
    out = ctypes.c_void_p()
    st = L.rk_ctx_create(0, 0, 2, None, None, ctypes.byref(out))   # uid NULL with 2 ranks
    assert st == librk.RK_EINVAL
    assert b"uid" in L.rk_last_error()


def test_struct_layouts(librk):
    # rk_config: method,m,k_max,k_keep,select_count,ortho,trunc (7 ints) + rk_precond (32 B:
    # 2 ints, 2 doubles, zblocks + padding; 8-aligned at 32) + tol + max_matvecs + divergence
    assert ctypes.sizeof(librk.rk_precond) == 32
    assert librk.rk_config.pc.offset == 32
    assert ctypes.sizeof(librk.rk_config) == 88
    assert ctypes.sizeof(librk.rk_report) == 72
    assert ctypes.sizeof(librk.rk_grid) == 48


def test_abi_struct_sizes_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "rk.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(rk_config), sizeof(rk_report),'
                   ' sizeof(rk_grid), sizeof(rk_precond), offsetof(rk_config, pc));return 0;}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    assert out == ["88", "72", "48", "32", "32"]


def test_product_does_not_import_oracle():
    """The product package never imports the oracle (DESIGN.md boundary)."""
    pkg = os.path.join(ROOT, "paper_1501_03358_b200")
    for dp, _, fs in os.walk(pkg):
        for f in fs:
            if f.endswith((".py", ".cpp", ".cu", ".h")):
                txt = open(os.path.join(dp, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, re.M), f
