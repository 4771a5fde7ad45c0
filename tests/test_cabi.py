"""The C-ABI library loads and exports every symbol include/dnnmg_b200.h declares
(no compute calls: runs without a GPU)."""
import os
import re
import subprocess

from paper_2307_14837_b200 import _lib

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "dnnmg_b200.h")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int32_t|const char\*)\s+(dnnmg_\w+)\s*\(", src, re.M)))


def test_header_declares_the_api():
    names = declared()
    for n in ("dnnmg_prolongate", "dnnmg_residual", "dnnmg_gather", "dnnmg_mlp_forward",
              "dnnmg_scatter_update", "dnnmg_correction_step"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for n in declared():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\b(dnnmg_\w+)\b", out))
    assert set(declared()) <= exported
    assert set(_lib.EXPORTS) <= exported
    # and the ctypes binding (the reference-side stub of INTEGRATION.md) covers all of them
    assert set(declared()) <= set(_lib.EXPORTS)


def test_status_strings_and_version():
    lib = _lib.load()
    assert lib.dnnmg_version() >= 100
    assert lib.dnnmg_status_string(0) == b"ok"
    assert b"architecture" in lib.dnnmg_status_string(4)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
