"""ctypes binding of libdnnmg_b200.so (C ABI in include/dnnmg_b200.h).

The shared library is the product: there is no Python/numpy fallback for any
compute call.  If the library is missing or no CUDA device is present, every
compute entry point raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdnnmg_b200.so")

DNNMG_OK, DNNMG_ERR_ARG, DNNMG_ERR_CUDA, DNNMG_ERR_UNSUPPORTED, DNNMG_ERR_ARCH = range(5)
ACT_RELU, ACT_TANH = 0, 1
PREC_FP32, PREC_BF16, PREC_TF32X3, PREC_F16X3, PREC_FP8 = 0, 1, 2, 3, 4
PRECISIONS = {"fp32": PREC_FP32, "bf16": PREC_BF16, "tf32x3": PREC_TF32X3, "f16x3": PREC_F16X3,
              "fp8": PREC_FP8}
MAX_LAYERS = 16

c_i32, c_i64, c_f32, c_vp = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_void_p


class Prolong(ctypes.Structure):
    _fields_ = [("n_fine_nodes", c_i32), ("n_coarse_cells", c_i32),
                ("coarse_cell_nodes", c_vp), ("fine_src", c_vp), ("owner_ptr", c_vp),
                ("owner_node", c_vp), ("owner_code", c_vp), ("lat_node", c_vp)]


class Dirichlet(ctypes.Structure):
    _fields_ = [("n_nodes", c_i32), ("bc_code", c_vp), ("bc_values", c_vp),
                ("bc_code_owner", c_vp), ("lat_node_bc", c_vp)]


class Level(ctypes.Structure):
    _fields_ = [("n_nodes", c_i32), ("n_cells", c_i32), ("cell_nodes", c_vp), ("coords", c_vp),
                ("h_T", c_vp), ("node_cell_ptr", c_vp), ("node_cell_idx", c_vp),
                ("dof_mask", c_vp), ("geo_q", c_vp), ("node_order", c_vp),
                ("tc_const", c_vp), ("tc_geo", c_vp), ("tc_geo_affine", c_i32),
                ("visit_ptr", c_vp), ("visit_idx", c_vp), ("geo_box", c_vp)]


class Phys(ctypes.Structure):
    _fields_ = [("nu", c_f32), ("k", c_f32), ("alpha0", c_f32), ("delta0", c_f32),
                ("convection", c_i32)]


class PatchSet(ctypes.Structure):
    _fields_ = [("n_patches", c_i32), ("nodes_per_patch", c_i32), ("n_geo", c_i32),
                ("n_nodes", c_i32), ("node_table", c_vp), ("geom", c_vp),
                ("node_patch_ptr", c_vp), ("node_patch_idx", c_vp),
                ("tile_cap", c_i32), ("tile_nodes", c_vp), ("tile_count", c_vp), ("tile_slot", c_vp),
                ("node_order", c_vp), ("visit_ptr", c_vp), ("visit_idx", c_vp)]


class Mlp(ctypes.Structure):
    _fields_ = [("n_in", c_i32), ("n_hidden", c_i32), ("depth", c_i32), ("n_out", c_i32),
                ("activation", c_i32), ("precision", c_i32), ("W", c_vp * MAX_LAYERS),
                ("bn_scale", c_vp), ("bn_shift", c_vp), ("in_mean", c_vp), ("in_std", c_vp),
                ("packed", c_vp)]


class Restrict(ctypes.Structure):
    _fields_ = [("n_coarse_nodes", c_i32), ("n_fine_nodes", c_i32), ("ptr", c_vp), ("fine", c_vp),
                ("w", c_vp), ("n_coarse_cells", c_i32), ("coarse_cell_nodes", c_vp),
                ("owner_ptr", c_vp), ("owner_node", c_vp), ("owner_code", c_vp),
                ("node_cell_ptr", c_vp), ("node_cell_idx", c_vp), ("cell_scratch", c_vp)]


class Csr(ctypes.Structure):
    _fields_ = [("n_rows", c_i32), ("indptr", c_vp), ("indices", c_vp), ("data", c_vp)]


class Vanka(ctypes.Structure):
    _fields_ = [("n_cells", c_i32), ("ndl", c_i32), ("n_dofs", c_i32), ("cell_dofs", c_vp),
                ("dof_cell_ptr", c_vp), ("dof_cell_idx", c_vp), ("weight", c_vp), ("inv", c_vp)]


class HaloPlan(ctypes.Structure):
    _fields_ = [("n_nodes", c_i32), ("nodes", c_vp), ("n_send", c_i32), ("send", c_vp),
                ("merge_ptr", c_vp), ("merge_src", c_vp)]


class Slab(ctypes.Structure):
    _fields_ = [("peer", c_i32 * 2), ("cells", HaloPlan * 2), ("patches", HaloPlan * 2),
                ("send", c_vp * 2), ("recv", c_vp * 2)]


class StepBuffers(ctypes.Structure):
    _fields_ = [("x_tilde", c_vp), ("r", c_vp), ("elem", c_vp), ("X", c_vp), ("Y", c_vp),
                ("d", c_vp), ("x_mid", c_vp), ("mlp_ws", c_vp), ("mlp_ws_bytes", c_i64),
                ("b_ready", c_vp)]


EXPORTS = {
    "dnnmg_version": (c_i32, []),
    "dnnmg_status_string": (ctypes.c_char_p, [c_i32]),
    "dnnmg_last_error": (ctypes.c_char_p, []),
    "dnnmg_prolongate": (c_i32, [ctypes.POINTER(Prolong), c_vp, c_vp, ctypes.POINTER(Dirichlet), c_vp]),
    "dnnmg_apply_dirichlet": (c_i32, [ctypes.POINTER(Dirichlet), c_vp, c_vp]),
    "dnnmg_restrict": (c_i32, [ctypes.POINTER(Restrict), c_vp, c_vp, c_vp]),
    "dnnmg_level_geometry": (c_i32, [ctypes.POINTER(Level), c_vp, c_vp]),
    "dnnmg_level_geometry_box": (c_i32, [ctypes.POINTER(Level), c_vp, c_vp, c_vp]),
    "dnnmg_k2tc_constants_bytes": (c_i64, []),
    "dnnmg_k2tc_constants": (c_i32, [c_vp, c_vp]),
    "dnnmg_level_geometry_tc_floats": (c_i64, [ctypes.POINTER(Level), c_i32]),
    "dnnmg_level_geometry_tc": (c_i32, [ctypes.POINTER(Level), c_vp, c_i32, c_vp]),
    "dnnmg_stab": (c_i32, [ctypes.POINTER(Level), c_vp, ctypes.POINTER(Phys), c_vp, c_vp, c_vp]),
    "dnnmg_residual": (c_i32, [ctypes.POINTER(Level), c_vp, c_vp, c_vp, c_vp, ctypes.POINTER(Phys),
                               c_vp, c_vp, c_i32, c_vp]),
    "dnnmg_apply_operator": (c_i32, [ctypes.POINTER(Level), c_vp, c_vp, c_vp, ctypes.POINTER(Phys),
                                     c_vp, c_vp, c_vp]),
    "dnnmg_rhs_next": (c_i32, [ctypes.POINTER(Level), c_vp, ctypes.POINTER(Phys), c_vp, c_vp, c_vp]),
    "dnnmg_gather": (c_i32, [ctypes.POINTER(PatchSet), c_vp, c_vp, c_vp, c_vp]),
    "dnnmg_local_restrict": (c_i32, [ctypes.POINTER(PatchSet), c_vp, c_vp, c_vp]),
    "dnnmg_global_extend": (c_i32, [ctypes.POINTER(PatchSet), c_vp, c_vp, c_vp]),
    "dnnmg_mlp_packed_bytes": (c_i32, [ctypes.POINTER(Mlp), ctypes.POINTER(c_i64)]),
    "dnnmg_mlp_pack": (c_i32, [ctypes.POINTER(Mlp), c_vp, c_vp]),
    "dnnmg_mlp_forward": (c_i32, [ctypes.POINTER(Mlp), c_vp, c_i64, c_vp, c_vp]),
    "dnnmg_mlp_workspace_bytes": (c_i32, [ctypes.POINTER(Mlp), c_i64, ctypes.POINTER(c_i64)]),
    "dnnmg_mlp_forward_ws": (c_i32, [ctypes.POINTER(Mlp), c_vp, c_i64, c_vp, c_vp, c_i64, c_vp]),
    "dnnmg_mlp_forward_patches_ws": (c_i32, [ctypes.POINTER(Mlp), ctypes.POINTER(PatchSet), c_vp,
                                             c_vp, c_vp, c_vp, c_i64, c_vp]),
    "dnnmg_mlp_forward_patches": (c_i32, [ctypes.POINTER(Mlp), ctypes.POINTER(PatchSet), c_vp, c_vp,
                                          c_vp, c_vp]),
    "dnnmg_mlp_gather_mode": (c_i32, [ctypes.POINTER(Mlp), ctypes.POINTER(PatchSet)]),
    "dnnmg_scatter_update": (c_i32, [ctypes.POINTER(PatchSet), c_vp, c_vp, c_vp, c_f32, c_vp, c_vp,
                                     c_vp]),
    "dnnmg_dataset_rows": (c_i32, [ctypes.POINTER(PatchSet), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dnnmg_column_stats_scratch": (c_i32, [c_i32]),
    "dnnmg_ideal_update": (c_i32, [c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dnnmg_column_stats": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "dnnmg_vanka_setup": (c_i32, [c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dnnmg_vanka_smooth": (c_i32, [ctypes.POINTER(Vanka), ctypes.POINTER(Csr), c_vp, c_vp, c_i32,
                                   ctypes.c_double, c_vp, c_vp, c_vp]),
    "dnnmg_correction_step": (c_i32, [ctypes.POINTER(Prolong), c_i32, ctypes.POINTER(Dirichlet),
                                      ctypes.POINTER(Level), ctypes.POINTER(Phys),
                                      ctypes.POINTER(PatchSet), ctypes.POINTER(Mlp), c_vp, c_vp,
                                      c_f32, ctypes.POINTER(StepBuffers), c_vp, c_vp]),
    "dnnmg_correction_step_launches": (c_i32, [c_i32, ctypes.POINTER(Mlp)]),
    "dnnmg_halo_pack_rows": (c_i32, [ctypes.POINTER(HaloPlan), c_vp, c_vp, c_vp]),
    "dnnmg_halo_pack_patch_rows": (c_i32, [ctypes.POINTER(HaloPlan), ctypes.POINTER(PatchSet),
                                           c_vp, c_vp, c_vp]),
    "dnnmg_halo_merge_rows": (c_i32, [ctypes.POINTER(HaloPlan), c_vp, c_vp, c_vp, c_vp, c_vp,
                                      c_vp]),
    "dnnmg_halo_merge_scatter": (c_i32, [ctypes.POINTER(HaloPlan), ctypes.POINTER(PatchSet), c_vp,
                                         c_vp, c_vp, c_vp, c_f32, c_vp, c_vp, c_vp]),
    "dnnmg_nccl_available": (c_i32, []),
    "dnnmg_nccl_unique_id": (c_i32, [c_vp]),
    "dnnmg_nccl_comm_init": (c_i32, [c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "dnnmg_nccl_comm_count": (c_i32, [c_vp, ctypes.POINTER(c_i32)]),
    "dnnmg_nccl_comm_destroy": (c_i32, [c_vp]),
    "dnnmg_halo_exchange": (c_i32, [c_vp, ctypes.POINTER(c_i32), ctypes.POINTER(c_vp),
                                    ctypes.POINTER(c_vp), ctypes.POINTER(c_i64), c_vp]),
    "dnnmg_halo_pre": (c_i32, [ctypes.POINTER(Slab), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "dnnmg_halo_post": (c_i32, [ctypes.POINTER(Slab), c_vp, ctypes.POINTER(PatchSet), c_vp, c_vp,
                                c_vp, c_f32, c_vp, c_vp, c_vp]),
}

_lib = None


def load():
    """Load the shared library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not found: build it with `make` "
                               "(the CUDA library is required; there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(status, what=""):
    """Map a C status to the reference's exception types and messages."""
    if status == DNNMG_OK:
        return
    lib = load()
    detail = lib.dnnmg_last_error().decode()
    msg = f"{what}: {detail}" if what else detail
    if status in (DNNMG_ERR_ARG, DNNMG_ERR_ARCH):
        raise ValueError(msg)
    if status == DNNMG_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args), name)
