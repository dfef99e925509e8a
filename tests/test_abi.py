"""CPU-side checks of the C-ABI library: it builds, loads and exports every entry point that
include/msim.h declares (no compute calls: there is no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "msim.h")


def declared_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_[a-z_0-9]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for name in ["ms_create", "ms_destroy", "ms_upload_mesh", "ms_basis_upload", "ms_basis_build", "ms_timestep",
                 "ms_newton_step", "ms_pcg_solve", "ms_eval_elements", "ms_spmv", "ms_export_coarse"]:
        assert name in syms


def test_library_builds_and_exports_every_symbol():
    from paper_2508_13386_b200 import build
    lib_path = build.build(verbose=False)
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(ms_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(lib_path)
    for s in declared_symbols():
        assert hasattr(lib, s)


def test_binding_loads_and_reports_version():
    from paper_2508_13386_b200 import msim
    assert b"sm_100a" in msim.lib.ms_version()
    p = msim.default_params()
    assert abs(p.h - 1 / 60) < 1e-15 and p.ls_batch == 4 and p.max_newton == 100


def test_kernels_are_sm100a():
    from paper_2508_13386_b200 import build
    lib_path = build.build(verbose=False)
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
