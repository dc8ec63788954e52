"""ctypes binding of the C ABI declared in ``include/acr_b200.h``.

There is no CPU fallback: if the shared library cannot be loaded the
import fails loudly (``RuntimeError``).
"""

from __future__ import annotations

import ctypes as C
import os

from . import build as _build

_LIB = None

# (name, restype, argtypes)
_SIGS = [
    ("acr_plan_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                  C.c_int, C.POINTER(C.c_void_p)]),
    ("acr_plan_destroy", None, [C.c_void_p]),
    ("acr_nccl_unique_id", C.c_int, [C.c_void_p]),
    ("acr_plan_create_dist", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                       C.c_void_p, C.POINTER(C.c_void_p)]),
    ("acr_loopback_solve", C.c_int, [C.c_int, C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_int, C.c_int] + [C.c_void_p] * 6 +
     [C.c_int, C.c_void_p, C.POINTER(C.c_double)]),
    ("acr_plan_set_option", C.c_int, [C.c_void_p, C.c_int, C.c_longlong]),
    ("acr_factor", C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int, C.c_void_p]),
    ("acr_solve", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    ("acr_factor_rhs", C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.c_int, C.c_void_p, C.c_int,
                                                                    C.c_void_p]),
    ("acr_solve_back", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    ("acr_levels", C.c_int, [C.c_void_p]),
    ("acr_cutoff_blocks", C.c_int, [C.c_void_p]),
    ("acr_tree_depths", C.c_int, [C.c_void_p]),
    ("acr_rank_profile", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int),
                                   C.POINTER(C.c_double)]),
    ("acr_storage_bytes", C.c_longlong, [C.c_void_p, C.c_int]),
    ("acr_device_bytes", C.c_longlong, [C.c_void_p]),
    ("acr_factor_ms", C.c_double, [C.c_void_p]),
    ("acr_solve_ms", C.c_double, [C.c_void_p]),
    ("acr_kernel_launches", C.c_longlong, [C.c_void_p]),
    ("acr_kernel_stats", C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_longlong),
                                   C.POINTER(C.c_double), C.POINTER(C.c_ulonglong)]),
    ("acr_last_error", C.c_int, [C.c_void_p, C.c_char_p, C.c_int]),
    ("acr_global_error", C.c_int, [C.c_char_p, C.c_int]),
    ("acr_block_to_dense", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int,
                                     C.c_void_p, C.c_void_p]),
    ("acr_residual", C.c_int, [C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 7 +
     [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_void_p]),
    ("acr_gen_constant", C.c_int, [C.c_int, C.c_int, C.POINTER(C.c_double)] +
     [C.c_void_p] * 6),
    ("acr_gen_varcoef", C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_longlong),
                                  C.POINTER(C.c_longlong), C.POINTER(C.c_double)] +
     [C.c_void_p] * 7),
    ("acr_gen_uniform", C.c_int, [C.POINTER(C.c_ulonglong), C.c_longlong, C.c_int,
                                  C.c_double, C.c_double, C.c_void_p, C.c_void_p]),
    ("acr_truncate_factor", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_void_p,
                                      C.c_void_p, C.c_double, C.c_int, C.c_void_p,
                                      C.c_void_p, C.POINTER(C.c_int), C.c_void_p]),
    ("acr_set_truncate_path", C.c_int, [C.c_int]),
    ("acr_block_export", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4 +
     [C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p]),
    ("acr_step_lift", C.c_int, [C.c_void_p] + [C.c_void_p] * 5 + [C.POINTER(C.c_int), C.c_void_p]),
    ("acr_step_reduce", C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p]),
    ("acr_step_rhs", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
    ("acr_step_backsub", C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                   C.c_void_p, C.c_void_p]),
    ("acr_step_info", C.c_int, [C.c_void_p, C.c_int, C.c_int] + [C.POINTER(C.c_int)] * 4),
    ("acr_step_export", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5),
    ("acr_step_free", C.c_int, [C.c_void_p, C.c_int]),
    ("acr_leaf_inverse", C.c_int, [C.c_int, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_int), C.c_void_p]),
]

EXPORTED = [s[0] for s in _SIGS]

ACR_OK, ACR_EARG, ACR_ESINGULAR, ACR_ECUDA, ACR_EINTERNAL = range(5)


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load (building first if needed and nvcc is present) the library."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("ACR_LIB_OVERRIDE") or _build.LIB   # A/B development aid
    if path == _build.LIB and build_if_missing and (not os.path.exists(path) or _build.needs_build()) \
            and os.path.exists(_build.NVCC):
        _build.build()
    if not os.path.exists(path):
        raise RuntimeError(
            f"ACR CUDA library not found at {path}; run "
            "`python -m paper_1604_00617_b200.build` (no CPU fallback exists)")
    lib = C.CDLL(path)
    for name, res, args in _SIGS:
        if path != _build.LIB and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def last_error(plan=None) -> str:
    lib = load()
    buf = C.create_string_buffer(1024)
    if plan:
        lib.acr_last_error(plan, buf, 1024)
    else:
        lib.acr_global_error(buf, 1024)
    return buf.value.decode(errors="replace")
