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


def test_f16x3_rejects_unbounded_activation():
    """f16x3 splits activations into fp16 parts: the C ABI refuses it for relu models
    (host-side check, no GPU needed), and the Python layer runs them in tf32x3."""
    import ctypes
    from paper_2307_14837_b200.net import effective_precision
    lib = _lib.load()
    dummy = ctypes.c_void_p(16)          # never dereferenced by the host-side checks
    W = (ctypes.c_void_p * _lib.MAX_LAYERS)(*([16] * 4 + [0] * (_lib.MAX_LAYERS - 4)))
    for act, want in ((_lib.ACT_RELU, 3), (_lib.ACT_TANH, 0)):
        m = _lib.Mlp(240, 256, 3, 81, act, _lib.PRECISIONS["f16x3"], W, dummy, dummy, dummy,
                     dummy, None)
        nbytes = ctypes.c_int64(-1)
        assert lib.dnnmg_mlp_packed_bytes(ctypes.byref(m), ctypes.byref(nbytes)) == want
        if want:
            assert b"f16x3" in lib.dnnmg_last_error()
        else:
            assert nbytes.value > 0
    assert effective_precision("relu", "f16x3") == "tf32x3"
    assert effective_precision("tanh", "f16x3") == "f16x3"
    assert effective_precision("relu", "bf16") == "bf16"


def test_layered_workspace_size_is_checked():
    """A workspace smaller than dnnmg_mlp_workspace_bytes(m, n_rows) is an argument error,
    not a silent overrun (host-side check before any launch)."""
    import ctypes
    lib = _lib.load()
    dummy = ctypes.c_void_p(256)
    W = (ctypes.c_void_p * _lib.MAX_LAYERS)(*([256] * 4 + [0] * (_lib.MAX_LAYERS - 4)))
    m = _lib.Mlp(174, 64, 3, 81, _lib.ACT_TANH, _lib.PRECISIONS["tf32x3"], W, dummy, dummy,
                 dummy, dummy, dummy)
    need = ctypes.c_int64(0)
    rows = 5000
    assert lib.dnnmg_mlp_workspace_bytes(ctypes.byref(m), rows, ctypes.byref(need)) == 0
    assert need.value > 0
    rc = lib.dnnmg_mlp_forward_ws(ctypes.byref(m), dummy, rows, dummy, dummy, need.value - 1,
                                  None)
    assert rc == 1 and b"workspace" in lib.dnnmg_last_error()


def test_ctypes_structs_match_the_header(tmp_path):
    """The ctypes mirror of every C-ABI struct (paper_2307_14837_b200/_lib.py, the binding a
    reference maintainer would write) has the size and the field offsets a C compiler gives
    include/dnnmg_b200.h: a field appended on one side only would shift every later one."""
    import ctypes
    pairs = {"dnnmg_prolong_t": _lib.Prolong, "dnnmg_restrict_t": _lib.Restrict,
             "dnnmg_dirichlet_t": _lib.Dirichlet, "dnnmg_level_t": _lib.Level,
             "dnnmg_phys_t": _lib.Phys, "dnnmg_patchset_t": _lib.PatchSet,
             "dnnmg_mlp_t": _lib.Mlp, "dnnmg_csr_t": _lib.Csr, "dnnmg_vanka_t": _lib.Vanka,
             "dnnmg_step_buffers_t": _lib.StepBuffers, "dnnmg_halo_plan_t": _lib.HaloPlan,
             "dnnmg_slab_t": _lib.Slab}
    src = open(HEADER).read()
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "dnnmg_b200.h"',
             'int main(void) {']
    fields = {}
    for cname in pairs:
        body = re.search(r"typedef struct \{([^{}]*)\}\s*" + cname + ";",
                         re.sub(r"/\*.*?\*/", "", src, flags=re.S)).group(1)
        names = [re.search(r"(\w+)\s*(?:\[[^\]]*\])?\s*$", part.strip()).group(1)
                 for d in body.split(";") if d.strip() for part in d.split(",")]
        fields[cname] = names
        lines.append(f'  printf("{cname} %zu", sizeof({cname}));')
        for f in names:
            lines.append(f'  printf(" %zu", offsetof({cname}, {f}));')
        lines.append('  printf("\\n");')
    lines += ['  return 0;', '}']
    c = tmp_path / "layout.c"
    c.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(c), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    for row in out.strip().splitlines():
        cname, size, *offs = row.split()
        cls = pairs[cname]
        assert ctypes.sizeof(cls) == int(size), cname
        assert [f for f, _ in cls._fields_] == fields[cname], cname
        assert [getattr(cls, f).offset for f, _ in cls._fields_] == [int(o) for o in offs], cname
