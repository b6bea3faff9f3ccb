"""ctypes mirror of include/xyzb.h (the C ABI of libxyzb.so).

Struct layouts here must match include/xyzb.h field for field; the
`xyzb_abi_version()` check in `_lib.load()` guards against drift.
"""
from __future__ import annotations

import ctypes as C

ABI_VERSION = 3

OK, E_DATA, E_GUARD, E_SOLVER, E_CUDA, E_INTERNAL = 0, 3, 4, 5, 10, 11
MODE_BINARY, MODE_CONTINUOUS_Y, MODE_CONTINUOUS_XY = 0, 1, 2
TOPK_HITS, TOPK_CANDIDATES = 0, 1
TRANSFORM_NONE, TRANSFORM_SIGN, TRANSFORM_UNBIASED = 0, 1, 2
NUM_STAGES = 8
STAGE_NAMES = ("draws", "project", "sort", "join", "verify", "merge", "estimate", "other")


class Problem(C.Structure):
    _fields_ = [
        ("n_rows", C.c_uint64),
        ("n_cols", C.c_uint64),
        ("x_words", C.POINTER(C.c_uint64)),
        ("x_real", C.POINTER(C.c_double)),
        ("device", C.c_int32),
        ("flags", C.c_int32),
        ("x_real32", C.POINTER(C.c_float)),
        ("devices", C.POINTER(C.c_int32)),
        ("n_devices", C.c_uint64),
    ]


class Response(C.Structure):
    _fields_ = [
        ("y_sign", C.POINTER(C.c_int8)),
        ("y_real", C.POINTER(C.c_double)),
    ]


class Params(C.Structure):
    _fields_ = [
        ("m", C.c_uint64),
        ("l", C.c_uint64),
        ("gamma", C.c_double),
        ("mode", C.c_int32),
        ("transform", C.c_int32),
        ("search_negatives", C.c_int32),
        ("stop_after_first_hit", C.c_int32),
        ("estimate_complexity", C.c_int32),
        ("threads", C.c_int32),
        ("seed", C.c_uint64),
        ("max_candidates_per_rep", C.c_uint64),
        ("strength_sample_size", C.c_uint64),
        ("top_k", C.c_uint64),
        ("rep_begin", C.c_uint64),
        ("rep_end", C.c_uint64),
        ("top_k_mode", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Hit(C.Structure):
    _fields_ = [
        ("j", C.c_uint32),
        ("k", C.c_uint32),
        ("strength", C.c_double),
        ("found_at_repetition", C.c_uint32),
        ("sign", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("hits", C.POINTER(Hit)),
        ("n_hits", C.c_uint64),
        ("order_keys", C.POINTER(C.c_uint64)),
        ("top_k", C.POINTER(C.c_uint64)),
        ("n_top_k", C.c_uint64),
        ("repetitions_run", C.c_uint64),
        ("candidates_checked", C.c_uint64),
        ("candidates_enumerated", C.c_uint64),
        ("aborted_repetitions", C.c_uint64),
        ("wall_time_s", C.c_double),
        ("estimated_c", C.c_double),
        ("gamma0", C.c_double),
        ("m_used", C.c_uint64),
        ("l_used", C.c_uint64),
        ("runs_executed", C.c_uint64),
        ("verified_pairs", C.c_uint64),
        ("device_ms", C.c_double),
        ("stage_ms", C.c_double * NUM_STAGES),
        ("stage_bytes", C.c_uint64 * NUM_STAGES),
        ("stage_launches", C.c_uint64 * NUM_STAGES),
        ("kernel_launches", C.c_uint64),
        ("verify_kernel_ms", C.c_double),
        ("verify_launches", C.c_uint64),
        ("gamma_effective", C.c_double),
        ("devices_used", C.c_uint64),
        ("attempts", C.c_uint64),
    ]


class ScoredPair(C.Structure):
    _fields_ = [
        ("j", C.c_uint32),
        ("k", C.c_uint32),
        ("strength", C.c_double),
    ]


ERRBUF = 1024


def errbuf():
    return C.create_string_buffer(ERRBUF)


# Every symbol include/xyzb.h declares, with (restype, argtypes).
_P = C.c_void_p
SIGNATURES = {
    "xyzb_abi_version": (C.c_int, []),
    "xyzb_params_init": (None, [C.POINTER(Params)]),
    "xyzb_device_count": (C.c_int, []),
    "xyzb_dataset_create": (C.c_int, [C.POINTER(Problem), C.POINTER(_P), C.c_char_p, C.c_size_t]),
    "xyzb_dataset_destroy": (None, [_P]),
    "xyzb_dataset_open": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(_P), C.c_char_p, C.c_size_t]),
    "xyzb_dataset_shape": (C.c_int, [_P, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_int32)]),
    "xyzb_search": (C.c_int, [_P, C.POINTER(Response), C.POINTER(Params), C.POINTER(C.c_uint32),
                              C.POINTER(Result), C.c_char_p, C.c_size_t]),
    "xyzb_merge_results": (C.c_int, [_P, C.POINTER(Result), C.c_uint64, C.POINTER(Params),
                                     C.POINTER(Result), C.c_char_p, C.c_size_t]),
    "xyzb_result_free": (None, [C.POINTER(Result)]),
    "xyzb_project_keys": (C.c_int, [_P, C.POINTER(C.c_uint32), C.c_uint64, C.c_uint64,
                                    C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "xyzb_equal_pairs": (C.c_int, [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.c_uint64, C.c_int32,
                                   C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
    "xyzb_pair_strengths": (C.c_int, [_P, C.POINTER(Response), C.POINTER(Params), C.POINTER(C.c_uint32),
                                      C.c_uint64, C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "xyzb_pair_agreements": (C.c_int, [_P, _P, C.POINTER(C.c_uint32), C.c_uint64, C.POINTER(C.c_uint64), C.c_char_p,
                                       C.c_size_t]),
    "xyzb_brute_force": (C.c_int, [_P, C.POINTER(C.c_int8), C.c_int32, C.c_double, C.c_int32, C.c_uint64,
                                   C.c_uint64, C.c_int32, C.POINTER(C.POINTER(ScoredPair)), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64), C.POINTER(C.POINTER(C.c_uint64)), C.c_char_p,
                                   C.c_size_t]),
    "xyzb_brute_force_weighted": (C.c_int, [_P, C.POINTER(C.c_double), C.c_int32, C.c_double, C.c_int32, C.c_uint64,
                                            C.c_uint64, C.c_int32, C.POINTER(C.POINTER(ScoredPair)),
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                            C.POINTER(C.POINTER(C.c_uint64)), C.c_char_p, C.c_size_t]),
    "xyzb_design_create": (C.c_int, [C.POINTER(C.c_double), C.c_uint64, C.c_uint64, C.POINTER(C.c_double), C.c_int32,
                                     C.POINTER(_P), C.c_char_p, C.c_size_t]),
    "xyzb_design_destroy": (None, [_P]),
    "xyzb_design_main_correlations": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_char_p,
                                                C.c_size_t]),
    "xyzb_design_pair_correlations": (C.c_int, [_P, C.POINTER(C.c_double), C.POINTER(C.c_uint32), C.c_uint64,
                                                C.POINTER(C.c_double), C.c_char_p, C.c_size_t]),
    "xyzb_free": (None, [_P]),
}


def bind(lib, signatures):
    for name, (res, args) in signatures.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib
