"""The C-ABI library loads on CPU and exports every symbol include/*.h declares."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2601_07508_b200 as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fpmm_b200.h")).read()
    return sorted(set(re.findall(r"\b(fpmm_b200_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol():
    lib = ctypes.CDLL(F.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_sm100a_only_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        return
    assert "sm_100a" in out.stdout
    assert not re.search(r"sm_(?!100a)\d+", out.stdout)


def test_dmma_and_tma_in_sass():
    out = subprocess.run(["cuobjdump", "-sass", F.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        return
    assert "DMMA.8x8x4" in out.stdout      # FP64 tensor-core MMA
    assert "UBLKCP.S.G" in out.stdout      # TMA bulk copy global -> shared


def test_version_and_errors():
    assert F.lib().fpmm_b200_version() == 1
    try:
        F.word_base(1, 2)
    except F.Error as e:
        assert "p must exceed 1" in str(e)
    else:
        raise AssertionError("expected Error")


def test_cpp_shim_compiles_and_runs_host_rules(tmp_path):
    """The C++ drop-in header (include/fpmm_b200/fpmm.hpp) against the library."""
    src = os.path.join(ROOT, "tests", "cpp", "shim_rules.cpp")
    exe = tmp_path / "shim_rules"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", str(exe),
                    F.LIB_PATH, "-Wl,-rpath," + os.path.dirname(F.LIB_PATH)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True)
    assert "OK" in out.stdout


@pytest.mark.gpu
def test_cpp_shim_product_on_gpu(tmp_path):
    """A reference-style C++ program against the drop-in header runs every
    engine and product variant on the GPU and matches exact dot products."""
    src = os.path.join(ROOT, "tests", "cpp", "shim_product.cpp")
    exe = tmp_path / "shim_product"
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), src, "-o", str(exe),
                    F.LIB_PATH, "-Wl,-rpath," + os.path.dirname(F.LIB_PATH)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "OK" in out.stdout, out.stdout + out.stderr
