"""ctypes binding of libtnc.so (include/tnc.h).

This is the binding a maintainer would add to the reference package to route
``tnsim`` amplitude evaluation through the B200 engine.
Loading never silently degrades: if the shared library is missing or no sm_100
device is present, ``lib()`` / ``require_device()`` raise.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

MAX_LEGS = 40
MAX_CUTS = 16
C64, C128 = 0, 1
K_AUTO, K_GENERIC, K_SKINNY, K_TC = 0, 1, 2, 3

LIB_PATH = Path(__file__).with_name("libtnc.so")

# symbols declared in include/tnc.h (checked by tests/test_abi.py)
EXPORTS = (
    "tnc_version", "tnc_struct_size", "tnc_device_check", "tnc_last_error",
    "tnc_project", "tnc_step", "tnc_slice_sum", "tnc_contract_path",
    "tnc_contract_pair_workspace", "tnc_contract_pair",
    "tnc_pair_plan_create", "tnc_pair_plan_execute", "tnc_pair_plan_kernel", "tnc_pair_plan_destroy",
)


class NativeError(RuntimeError):
    """A libtnc entry point returned an error code."""


class Site(C.Structure):
    _fields_ = [
        ("ptr", C.c_void_p), ("sel", C.c_void_p), ("zstride", C.c_int64), ("vstride", C.c_int64),
        ("nvariants", C.c_int64), ("ncut", C.c_int32), ("_pad", C.c_int32),
        ("cut_stride", C.c_int64 * MAX_CUTS), ("cut_div", C.c_int64 * MAX_CUTS),
        ("cut_ext", C.c_int64 * MAX_CUTS),
    ]


class StepDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("kernel", C.c_int32), ("Z", C.c_int64), ("slices_per_b", C.c_int64),
        ("s0", C.c_int64), ("acc", C.c_void_p), ("acc_zstride", C.c_int64),
        ("out", C.c_void_p), ("out_zstride", C.c_int64), ("site", Site),
        ("M", C.c_int64), ("nf", C.c_int32), ("c_n_contig", C.c_int32),
        ("f_dim", C.c_int64 * MAX_LEGS), ("f_astride", C.c_int64 * MAX_LEGS),
        ("f_cstride", C.c_int64 * MAX_LEGS), ("K", C.c_int64), ("N", C.c_int64),
        ("a_koff", C.c_void_p), ("b_koff", C.c_void_p), ("b_noff", C.c_void_p), ("c_noff", C.c_void_p),
        ("a_rows_contig", C.c_int32), ("c_rows_contig", C.c_int32), ("b_dense", C.c_int32),
        ("conj_b", C.c_int32), ("amax_out", C.c_void_p), ("amax_in", C.c_void_p),
        ("nn", C.c_int32), ("_pad2", C.c_int32),
        ("n_dim", C.c_int64 * MAX_LEGS), ("n_cstride", C.c_int64 * MAX_LEGS),
    ]


class ProjectDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("conj", C.c_int32), ("Z", C.c_int64), ("slices_per_b", C.c_int64),
        ("s0", C.c_int64), ("site", Site), ("out", C.c_void_p), ("out_zstride", C.c_int64),
        ("nd", C.c_int32), ("_pad", C.c_int32),
        ("dim", C.c_int64 * MAX_LEGS), ("src_stride", C.c_int64 * MAX_LEGS),
    ]


class SliceSumDesc(C.Structure):
    _fields_ = [
        ("dtype", C.c_int32), ("accumulate", C.c_int32), ("B", C.c_int64), ("slices_per_b", C.c_int64),
        ("x", C.c_void_p), ("x_zstride", C.c_int64), ("amp", C.c_void_p),
    ]


class PathDesc(C.Structure):
    _fields_ = [
        ("first", ProjectDesc), ("nsteps", C.c_int32), ("_pad", C.c_int32),
        ("steps", C.POINTER(StepDesc)), ("reduce", SliceSumDesc),
    ]


_LIB = None


def lib():
    """Load libtnc.so (built by __graft_entry__.build()); raises if absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = os.environ.get("TNC_LIB", str(LIB_PATH))
    if not Path(path).exists():
        raise NativeError(f"libtnc.so not found at {path}; run __graft_entry__.build()")
    L = C.CDLL(path)
    L.tnc_version.restype = C.c_int
    L.tnc_struct_size.restype = C.c_size_t
    L.tnc_struct_size.argtypes = [C.c_int]
    L.tnc_device_check.restype = C.c_int
    L.tnc_last_error.restype = C.c_char_p
    for name, desc in (("tnc_project", ProjectDesc), ("tnc_step", StepDesc),
                       ("tnc_slice_sum", SliceSumDesc), ("tnc_contract_path", PathDesc)):
        fn = getattr(L, name)
        fn.restype = C.c_int
        fn.argtypes = [C.POINTER(desc), C.c_void_p]
    L.tnc_contract_pair_workspace.restype = C.c_size_t
    L.tnc_contract_pair_workspace.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.tnc_contract_pair.restype = C.c_int
    L.tnc_contract_pair.argtypes = [
        C.c_int, C.c_int64,
        C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
        C.c_void_p, C.c_int, C.c_void_p, C.c_int64,
        C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
        C.c_void_p, C.c_int64, C.c_void_p, C.c_size_t, C.c_void_p,
    ]
    L.tnc_pair_plan_create.restype = C.c_int
    L.tnc_pair_plan_create.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_int,
                                       C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
    L.tnc_pair_plan_execute.restype = C.c_int
    L.tnc_pair_plan_execute.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                        C.c_void_p, C.c_int64, C.c_void_p]
    L.tnc_pair_plan_kernel.restype = C.c_int
    L.tnc_pair_plan_kernel.argtypes = [C.c_void_p]
    L.tnc_pair_plan_destroy.restype = None
    L.tnc_pair_plan_destroy.argtypes = [C.c_void_p]
    for i, cls in enumerate((Site, StepDesc, ProjectDesc, SliceSumDesc, PathDesc)):
        native = L.tnc_struct_size(i)
        if native != C.sizeof(cls):
            raise NativeError(f"ABI mismatch for {cls.__name__}: C {native} vs ctypes {C.sizeof(cls)}")
    _LIB = L
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = lib().tnc_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def require_device() -> None:
    check(lib().tnc_device_check(), "tnc_device_check")
