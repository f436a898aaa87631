"""ctypes binding of the C ABI in include/chebm2l.h (libchebm2l.so, sm_100a).

There is no CPU fallback: importing the product path without the built
library, or calling it on a machine without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libchebm2l.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

CFM_OK = 0
CFM_ERR_VALUE = 1
CFM_ERR_PRECOMPUTE = 2
CFM_ERR_BUDGET = 3
CFM_ERR_CUDA = 4
CFM_ERR_INTERNAL = 5

VARIANT_IDS = {"na": 0, "nasym": 1, "nablk": 2, "sa": 3, "sarcmp": 4, "ia": 5, "iasym": 6, "iablk": 7}

# Every symbol include/chebm2l.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "cfm_last_error",
    "cfm_abi_version",
    "cfm_handler_create",
    "cfm_handler_destroy",
    "cfm_set_dense_group",
    "cfm_set_lowrank_group",
    "cfm_set_shared_group",
    "cfm_set_level",
    "cfm_apply_level_csr",
    "cfm_plan_level_cells",
    "cfm_plan_level_csr",
    "cfm_plan_level_cells_subset",
    "cfm_apply_planned",
    "cfm_apply_levels",
    "cfm_plan_stats",
    "cfm_plan_info",
    "cfm_plan_two_stage",
    "cfm_classify_count",
    "cfm_classify_fill",
    "cfm_classify_count_device",
    "cfm_classify_fill_device",
    "cfm_last_apply_stats",
    "cfm_tree_build",
    "cfm_tree_level_size",
    "cfm_tree_level_cells",
    "cfm_tree_leaf_particles",
    "cfm_tree_destroy",
    "cfm_fmm_create",
    "cfm_fmm_destroy",
    "cfm_fmm_p2m",
    "cfm_fmm_m2m",
    "cfm_fmm_l2l",
    "cfm_fmm_l2p",
    "cfm_fmm_p2p",
    "cfm_assemble_operators",
    "cfm_last_csr_plan_info",
    "cfm_classify_targets_count",
    "cfm_classify_targets_fill",
    "cfm_gather_rows",
    "cfm_aca_batch",
)

# libcfm_batch.so (include/chebm2l_batch.h): the reference batch -> CSR in C.
BATCH_LIB_NAME = "libcfm_batch.so"
BATCH_EXPORTS = ("cfm_batch_count", "cfm_batch_fill", "cfm_flush_sequence")

_P = ctypes.c_void_p
_I = ctypes.c_int
_I64 = ctypes.c_int64
_D = ctypes.c_double

_SIGS = {
    "cfm_last_error": ([], ctypes.c_char_p),
    "cfm_abi_version": ([], _I),
    "cfm_handler_create": ([_I, _I, _I, _I, ctypes.POINTER(_P)], _I),
    "cfm_handler_destroy": ([_P], _I),
    "cfm_set_dense_group": ([_P, _I, _I, _P, _I, _P, _P], _I),
    "cfm_set_lowrank_group": ([_P, _I, _I, _P, _I, _P, _P, _P, _P], _I),
    "cfm_set_shared_group": ([_P, _I, _I, _I, _P, _P, _I, _P, _P, _P], _I),
    "cfm_set_level": ([_P, _I, _I, _D], _I),
    "cfm_apply_level_csr": ([_P, _I, _I64, _P, _P, _P, _P, _I, _P, _I64, _P, _P, _P], _I),
    "cfm_plan_level_cells": ([_P, _I, _I64, _P, _I, _P, _P], _I),
    "cfm_plan_level_csr": ([_P, _I, _I64, _P, _P, _P, _P, _I, _I64, _P], _I),
    "cfm_plan_level_cells_subset": ([_P, _I, _I64, _P, _I64, _P, _I, _P, _P, _P, _P], _I),
    "cfm_apply_planned": ([_P, _I, _P, _I64, _P, _P], _I),
    "cfm_apply_levels": ([_P, _I, _P, _P, _P, _P, _P], _I),
    "cfm_plan_stats": ([_P, _I, _P, _P, _P, _P, _P, _P], _I),
    "cfm_plan_info": ([_P, _I, _P, _P], _I),
    "cfm_plan_two_stage": ([_P, _I, _P], _I),
    "cfm_classify_count": ([_I, _I, _I64, _P, _P, _P], _I),
    "cfm_classify_fill": ([_I, _I, _I64, _P, _P, _P, _P, _P, _P], _I),
    "cfm_classify_count_device": ([_I, _I, _I64, _P, _P, _P, _P], _I),
    "cfm_classify_fill_device": ([_I, _I, _I64, _P, _P, _P, _P, _P], _I),
    "cfm_last_apply_stats": ([_P, _P, _P], _I),
    "cfm_tree_build": ([_I, _P, _I64, _P, _D, _I, ctypes.POINTER(_P)], _I),
    "cfm_tree_level_size": ([_P, _I, _P], _I),
    "cfm_tree_level_cells": ([_P, _I, _P], _I),
    "cfm_tree_leaf_particles": ([_P, _P, _P], _I),
    "cfm_tree_destroy": ([_P], _I),
    "cfm_fmm_create": ([_P, _I, _P, ctypes.POINTER(_P)], _I),
    "cfm_fmm_destroy": ([_P], _I),
    "cfm_fmm_p2m": ([_P, _P, _I, _P, _P], _I),
    "cfm_fmm_m2m": ([_P, _I, _P, _P, _I, _P], _I),
    "cfm_fmm_l2l": ([_P, _I, _P, _P, _I, _P], _I),
    "cfm_fmm_l2p": ([_P, _P, _I, _P, _P], _I),
    "cfm_fmm_p2p": ([_P, _I, _D, _P, _I, _P, _I, _P], _I),
    "cfm_assemble_operators": ([_I, _I, _D, _I, _P, _D, _I, _P, _P, _P], _I),
    "cfm_last_csr_plan_info": ([_P, _P, _P, _P, _P], _I),
    "cfm_classify_targets_count": ([_I, _I, _I64, _P, _I64, _P, _P, _P], _I),
    "cfm_classify_targets_fill": ([_I, _I, _I64, _P, _I64, _P, _P, _P, _P], _I),
    "cfm_gather_rows": ([_I, _P, _I64, _P, _I64, _P, _P], _I),
    "cfm_aca_batch": ([_I, _I, _I, _I, _P, _D, _I, _P, _P, _P, _P, _P], _I),
}

_lib = None


class NativeError(RuntimeError):
    """A CUDA/internal failure reported through the C ABI."""


def load(path: str | os.PathLike | None = None):
    """Load libchebm2l.so (raises if it was not built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # CFM_LIB_PATH: load another build of the library (A/B timing experiments)
    p = Path(path) if path is not None else Path(os.environ.get("CFM_LIB_PATH", LIB_PATH))
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build the CUDA extension first (python -c "
            "'import __graft_entry__ as g; g.build()' or `make`)"
        )
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGS.items():
        if "CFM_LIB_PATH" in os.environ and not hasattr(lib, name):
            continue  # an older experimental build
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


_batch_lib = None


def load_batch():
    """Load libcfm_batch.so with ctypes.PyDLL (the GIL stays held during its
    calls, which read the caller's Python objects)."""
    global _batch_lib
    if _batch_lib is None:
        p = LIB_PATH.parent / BATCH_LIB_NAME
        if not p.exists():
            raise ImportError(f"{p} is missing: build the native extensions first (`make`)")
        lib = ctypes.PyDLL(str(p))
        lib.cfm_batch_count.argtypes = [ctypes.py_object, _P, _P, _P]
        lib.cfm_batch_count.restype = _I
        lib.cfm_batch_fill.argtypes = [ctypes.py_object, _P, _P, _P, _P, _I]
        lib.cfm_batch_fill.restype = _I
        lib.cfm_flush_sequence.argtypes = [_I64, _P, _P, _I, _I, _P, _P, _I64]
        lib.cfm_flush_sequence.restype = _I64
        _batch_lib = lib
    return _batch_lib


def check(rc: int, precompute_error=None, budget_error=None) -> None:
    """Map a C-ABI status to the reference's exception types."""
    if rc == CFM_OK:
        return
    msg = load().cfm_last_error().decode("utf-8", "replace")
    if rc == CFM_ERR_VALUE:
        raise ValueError(msg)
    if rc == CFM_ERR_PRECOMPUTE and precompute_error is not None:
        raise precompute_error(msg)
    if rc == CFM_ERR_BUDGET and budget_error is not None:
        raise budget_error(msg)
    raise NativeError(f"chebm2l error {rc}: {msg}")


def ptr(a) -> int | None:
    """Raw data pointer of a numpy array or a torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    data_ptr = getattr(a, "data_ptr", None)
    if data_ptr is not None:
        return int(data_ptr())
    raise TypeError(f"unsupported buffer type {type(a)!r}")
