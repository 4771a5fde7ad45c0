"""B200-native DNN-MG fine-level correction step (arXiv 2307.14837).

Drop-in for the correction path of the reference package ``dnnmg``: the
modules ``mesh``, ``space``, ``assembly``, ``net`` and ``patch_ops`` mirror the
reference names and signatures; their compute runs in the sm_100a kernels of
``libdnnmg_b200.so`` (C ABI: include/dnnmg_b200.h).  ``step.CorrectionStep`` is
the fused, device-resident production step.
"""

from . import mesh, elements, synthetic  # noqa: F401  (host-only modules)

__version__ = "0.1.0"


def library_path():
    from . import _lib
    return _lib.LIB_PATH
