"""The C-ABI library loads and exports every symbol include/scsf.h declares — CPU only.

No compute call is made (there is no GPU here); the library is built by
`paper_2510_23215_b200.build` (nvcc cross-compiles sm_100a without a GPU).
"""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "scsf.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(scsf_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2510_23215_b200 import build
    return build.build()


def test_header_declares_boundary():
    names = _declared()
    for required in ("scsf_sort", "scsf_solve_one", "scsf_solve_queue", "scsf_solve_chains"):
        assert required in names


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in _declared():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (scsf_\w+)", out))
    assert set(_declared()) <= exported


def test_abi_version_and_binding_table(libpath):
    from paper_2510_23215_b200 import scsf
    lib = scsf.load_library(libpath)
    assert lib.scsf_abi_version() == 2
    assert sorted(scsf.EXPORTED) == _declared()
    assert lib.scsf_launch_count() >= 0


def test_query_functions_without_gpu(libpath):
    from paper_2510_23215_b200 import scsf
    lib = scsf.load_library(libpath)
    assert lib.scsf_sort_workspace_bytes(1000, 2, 100, 1, 20) > 1000 * 1000 * 8
    ops = scsf.scsf_ops(2, 100, 100, 1, 1000, 0, 10016, 0)
    ws = lib.scsf_solve_workspace_bytes(ctypes.byref(ops), 100, 20)
    assert ws >= 4 * 120 * 10016 * 8
    assert lib.scsf_sort_workspace_bytes(0, 2, 100, 1, 20) == 0


def test_sass_uses_fp64_tensor_cores(libpath):
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    assert "DMMA" in out
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", libpath], capture_output=True, text=True).stdout


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2510_23215_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), fn


def test_new_queries_and_argument_errors_without_gpu(libpath):
    """Session-3 entry points: size queries and argument validation need no device."""
    from paper_2510_23215_b200 import scsf
    lib = scsf.load_library(libpath)
    ops = scsf.scsf_ops(2, 100, 100, 1, 10, 0, 10016, 1)
    assert lib.scsf_chain_state_doubles(ctypes.byref(ops), 100, 20) == 120 * (10000 + 1)
    assert lib.scsf_chain_state_doubles(ctypes.byref(ops), 0, 20) == 0
    assert lib.scsf_grf_workspace_bytes(100, 16) == 2 * 16 * 101 * 8
    # GRF: bad dim / K / family are rejected before any device work
    assert lib.scsf_grf_fields(4, 10, 4, 1.0, 0.5, 1.0, 0, 1, None, None, None, None, None, None, None, 0,
                               None) == scsf.SCSF_ERR_ARG
    assert lib.scsf_grf_fields(2, 10, 33, 1.0, 0.5, 1.0, 0, 1, None, None, None, None, None, None, None, 0,
                               None) == scsf.SCSF_ERR_ARG
    assert lib.scsf_grf_fields(2, 10, 4, 1.0, 0.5, 1.0, 7, 1, None, None, None, None, None, None, None, 0,
                               None) == scsf.SCSF_ERR_ARG
    # vibration assembly: the stencil kind must be VIB13 and the grid 2-D with nx, ny >= 3
    flux = scsf.scsf_ops(2, 8, 8, 1, 1, scsf.STENCIL_FLUX, 64, 1)
    assert lib.scsf_assemble_vibration(ctypes.byref(flux), 0.1, 1, 1, 64, 1, None) == scsf.SCSF_ERR_ARG
    vib3d = scsf.scsf_ops(3, 8, 8, 8, 1, scsf.STENCIL_VIB13, 512, 1)
    assert lib.scsf_assemble_vibration(ctypes.byref(vib3d), 0.1, 1, 1, 512, 1, None) == scsf.SCSF_ERR_ARG
    bad_kind = scsf.scsf_ops(2, 8, 8, 1, 1, 5, 64, 1)
    assert lib.scsf_solve_workspace_bytes(ctypes.byref(bad_kind), 4, 1) >= 0
    assert lib.scsf_assemble_vibration(ctypes.byref(bad_kind), 0.1, 1, 1, 64, 1, None) == scsf.SCSF_ERR_ARG


def test_library_has_no_undefined_internal_symbols():
    """Every scsf:: function the library calls is defined in it (a declaration that drifted from
    its definition would only fail at dlopen on the GPU box)."""
    import shutil
    import subprocess
    from paper_2510_23215_b200 import build as b
    nm = shutil.which("nm")
    if nm is None or not os.path.exists(b.LIB):
        pytest.skip("nm or libscsf.so missing")
    out = subprocess.run([nm, "-D", "--undefined-only", b.LIB], capture_output=True, text=True).stdout
    assert "scsf" not in out, [ln for ln in out.splitlines() if "scsf" in ln]
