"""Loader for the product library libxyzb.so (in-tree, built by
`make -C paper_1610_05108_b200/csrc` or `__graft_entry__.build()`).

There is no fallback: if the library is missing or no CUDA device is present,
every engine call raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxyzb.so")
SYNTH_PATH = os.path.join(HERE, "libxyzb_synth.so")


class XyzError(RuntimeError):
    code = _abi.E_INTERNAL


class DataError(XyzError):
    """xyz::data_error (errors.hpp:10-13)."""
    code = _abi.E_DATA


class GuardError(XyzError):
    """xyz::guard_error (errors.hpp:16-19)."""
    code = _abi.E_GUARD


class SolverError(XyzError):
    """xyz::solver_error (errors.hpp:22-25)."""
    code = _abi.E_SOLVER


class CudaError(XyzError):
    code = _abi.E_CUDA


class EngineError(XyzError):
    code = _abi.E_INTERNAL


_BY_CODE = {c.code: c for c in (DataError, GuardError, SolverError, CudaError, EngineError)}


def raise_for(code: int, err) -> None:
    if code == _abi.OK:
        return
    msg = err.value.decode(errors="replace") if err is not None else ""
    raise _BY_CODE.get(code, EngineError)(msg)


_lib = None
_synth = None


def load():
    """The bound libxyzb.so (raises if it is missing: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EngineError(f"{LIB_PATH} not built: run `make -C {os.path.join(HERE, 'csrc')}`")
        lib = _abi.bind(C.CDLL(LIB_PATH), _abi.SIGNATURES)
        if lib.xyzb_abi_version() != _abi.ABI_VERSION:
            raise EngineError("libxyzb.so ABI version mismatch with paper_1610_05108_b200/_abi.py")
        _lib = lib
    return _lib


TEST_OPTIONS = ("batch_entries", "hit_cap", "item_cap", "pair_cap", "grouping", "merge_large", "sign_verify_off",
                "trace", "brute_cuda")
GROUPING = {"auto": 0, "sort": 1, "part": 2, "msplit": 3}


def set_test_option(name: str, value: int) -> None:
    """xyzb_test_set_option (include/xyzb_testing.h): force a rare engine path
    in tests; 0 restores the default."""
    lib = load()
    fn = lib.xyzb_test_set_option
    fn.restype = C.c_int
    fn.argtypes = [C.c_char_p, C.c_longlong]
    if fn(name.encode(), int(value)) != 0:
        raise ValueError(f"unknown engine test option {name!r}")


_U64P = C.POINTER(C.c_uint64)
_U32P = C.POINTER(C.c_uint32)
_F64P = C.POINTER(C.c_double)
_I8P = C.POINTER(C.c_int8)

SYNTH_SIGNATURES = {
    "xyzb_synth_toy": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _U64P, _I8P]),
    "xyzb_synth_gwas": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, _U64P, _I8P, _U32P]),
    "xyzb_synth_gauss": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                   C.c_double, C.c_uint64, _F64P, _F64P, _U32P, _U32P]),
    "xyzb_synth_ar1": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64, C.c_double, C.c_uint64,
                                 _U64P, _I8P, _U32P]),
}


def load_synth():
    global _synth
    if _synth is None:
        if not os.path.exists(SYNTH_PATH):
            raise EngineError(f"{SYNTH_PATH} not built: run `make -C {os.path.join(HERE, 'csrc')}`")
        _synth = _abi.bind(C.CDLL(SYNTH_PATH), SYNTH_SIGNATURES)
    return _synth
