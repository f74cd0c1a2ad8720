"""CPU-side checks of the C-ABI boundary: the sm_100a library is built, loads,
and exports exactly the entry points include/confkv_b200.h declares (no
compute calls — this container has no GPU)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "confkv_b200.h"


def declared():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(ckv_\w+)\(", text, re.M)))


def _lib_path():
    from paper_2605_24786_b200 import build
    return build.build()


def test_header_declares_entry_points():
    names = declared()
    for n in ("ckv_create", "ckv_attend", "ckv_confidence", "ckv_manage", "ckv_step", "ckv_prefill",
              "ckv_stage_rows", "ckv_read_records", "ckv_read_cache", "ckv_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _lib_path()
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (ckv_\w+)", out))
    missing = set(declared()) - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"


def test_library_loads_and_binding_matches_header():
    lib_path = _lib_path()
    try:
        ctypes.CDLL(str(lib_path))
    except OSError as e:  # libcudart missing on a bare runner
        pytest.skip(f"cannot dlopen: {e}")
    from paper_2605_24786_b200 import _lib
    lib = _lib.load(lib_path)
    assert set(_lib.EXPORTED) == set(declared())
    assert lib.ckv_version() >= 100


def test_cubin_is_sm100a():
    lib = _lib_path()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
