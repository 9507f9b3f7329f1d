"""C-ABI checks that need no GPU: the in-tree sm_100a library loads, exports every entry
point include/sweep.h declares, and its host-side argument validation answers with the
documented status codes (no compute call is made)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sweep.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s*(sw_[a-z0-9_]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_1008_3699_b200 import build
    path = build.build()
    return ctypes.CDLL(path), path


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("sw_create_grid", "sw_decompose", "sw_sor_sweep", "sw_ilu0_factor", "sw_ilu_apply", "sw_pcg_solve",
              "sw_ssor_apply", "sw_residual_norm", "sw_destroy", "sw_last_error"):
        assert n in names, n


def test_library_exports_every_declared_symbol(lib):
    L, path = lib
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for n in declared_functions():
        assert n in exported, f"{n} declared in sweep.h but not exported by libsweep.so"
        assert getattr(L, n) is not None


def test_library_is_sm100a(lib):
    _, path = lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_validation_without_gpu(lib):
    L, _ = lib
    L.sw_last_error.restype = ctypes.c_char_p
    L.sw_create_grid.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                 ctypes.POINTER(ctypes.c_void_p)]
    h = ctypes.c_void_p(123)
    n = (ctypes.c_int64 * 3)(8, 8, 1)
    EINVAL = 1
    assert L.sw_create_grid(4, n, 0, 0.0, 0, ctypes.byref(h)) == EINVAL and h.value is None
    assert b"dim" in L.sw_last_error()
    bad = (ctypes.c_int64 * 3)(8, 0, 1)
    assert L.sw_create_grid(2, bad, 0, 0.0, 0, ctypes.byref(h)) == EINVAL
    assert L.sw_create_grid(2, n, 0, -1.0, 0, ctypes.byref(h)) == EINVAL
    assert L.sw_create_grid(2, n, 7, 0.0, 0, ctypes.byref(h)) == EINVAL
    assert L.sw_create_grid(2, n, 0, 0.0, 0, None) == EINVAL
    L.sw_decompose.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    assert L.sw_decompose(None, None, 0, 1) == EINVAL
    L.sw_destroy.argtypes = [ctypes.c_void_p]
    assert L.sw_destroy(None) == 0
    L.sw_launch_count.argtypes = [ctypes.c_void_p]
    L.sw_launch_count.restype = ctypes.c_int64
    assert L.sw_launch_count(None) == 0


def test_binding_fails_loudly_without_library(monkeypatch, tmp_path):
    from paper_1008_3699_b200 import binding
    monkeypatch.setattr(binding, "_lib", None)
    monkeypatch.setattr(binding, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(RuntimeError, match="missing"):
        binding.load()


def test_product_path_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_1008_3699_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, flags=re.M), f
                assert "oracle.c" not in txt and "liboracle" not in txt, f
