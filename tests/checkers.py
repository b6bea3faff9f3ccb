"""Loaders for the CHECKERS (test infrastructure, never the product path).

  oracle/liboracle.so        the CPU restatement of the parity contract
  oracle/_ref/libxyzref.so   the unmodified reference core (+ C harness)

Both are driven with the same plain structs as libxyzb.so (include/xyzb.h).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_1610_05108_b200 import _abi
from paper_1610_05108_b200.matrix import PackedMatrix, RealMatrix, make_problem, make_response
from paper_1610_05108_b200.report import SearchConfig, report_from_result

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libxyzref.so")

_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)
_U32P = C.POINTER(C.c_uint32)
_F64P = C.POINTER(C.c_double)

_ORACLE_SIGS = {
    "oracle_abi_version": (C.c_int, []),
    "oracle_search": (C.c_int, [C.POINTER(_abi.Problem), C.POINTER(_abi.Response), C.POINTER(_abi.Params),
                                C.POINTER(_abi.Result), C.c_char_p, C.c_size_t]),
    "oracle_result_free": (None, [C.POINTER(_abi.Result)]),
    "oracle_free": (None, [_P]),
    "oracle_draws": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int32, C.c_uint64, _F64P, _U32P,
                               C.c_char_p, C.c_size_t]),
    "oracle_project_keys": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, _U32P, C.c_uint64, C.c_uint64, _U64P,
                                      C.c_char_p, C.c_size_t]),
    "oracle_equal_pairs": (C.c_int, [_U64P, _U64P, C.c_uint64, C.POINTER(_U32P), _U64P, _U64P,
                                     C.c_char_p, C.c_size_t]),
    "oracle_pair_strengths": (C.c_int, [C.POINTER(_abi.Problem), C.POINTER(_abi.Response), C.c_int32, C.c_int32,
                                        _U32P, C.c_uint64, _F64P, C.c_char_p, C.c_size_t]),
}

_REF_SIGS = {
    "ref_abi_version": (C.c_int, []),
    "ref_search": (C.c_int, [C.POINTER(_abi.Problem), C.POINTER(_abi.Response), C.POINTER(_abi.Params),
                             C.POINTER(_abi.Result), C.c_char_p, C.c_size_t]),
    "ref_result_free": (None, [C.POINTER(_abi.Result)]),
    "ref_free": (None, [_P]),
    "ref_draw_subsample": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _F64P, _U64P,
                                     C.c_char_p, C.c_size_t]),
    "ref_project_keys": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, _U64P, C.c_uint64, _U64P, C.c_char_p, C.c_size_t]),
    "ref_build_z": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, C.POINTER(C.c_int8), _U64P, C.c_char_p, C.c_size_t]),
    "ref_equal_pairs": (C.c_int, [_U64P, _U64P, C.c_uint64, C.POINTER(_U32P), _U64P, _U64P, C.c_char_p, C.c_size_t]),
    "ref_pair_strengths": (C.c_int, [C.POINTER(_abi.Problem), C.POINTER(_abi.Response), C.c_int32, C.c_int32,
                                     _U32P, C.c_uint64, _F64P, C.c_char_p, C.c_size_t]),
    "ref_rademacher_matrix": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _U64P, C.c_char_p, C.c_size_t]),
    "ref_planted_instance": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_uint64,
                                       C.c_uint64, _U64P, C.POINTER(C.c_int8), C.c_char_p, C.c_size_t]),
    "ref_gaussian_matrix": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _F64P, C.c_char_p, C.c_size_t]),
    "ref_uniform_matrix": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, _F64P, C.c_char_p, C.c_size_t]),
    "ref_brute_force_topk": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, C.POINTER(C.c_int8), C.c_uint64, _U32P, _F64P,
                                       _U64P, C.c_char_p, C.c_size_t]),
    "ref_rescale_rows": (C.c_int, [_F64P, C.c_uint64, C.c_uint64, _F64P, _F64P, _F64P, C.c_char_p, C.c_size_t]),
    "ref_write_dataset": (C.c_int, [C.c_char_p, C.c_int32, _U64P, _F64P, C.c_uint64, C.c_uint64, C.c_char_p,
                                    C.c_size_t]),
    "ref_read_dataset": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), _U64P, _U64P, C.c_char_p, C.c_size_t]),
    "ref_brute_force_weighted": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, _F64P, C.c_int32, C.c_double,
                                           C.c_int32, C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(_U32P),
                                           C.POINTER(_F64P), _U64P, _U64P, C.POINTER(_U64P), C.c_char_p,
                                           C.c_size_t]),
    "ref_sample_strengths": (C.c_int, [C.POINTER(_abi.Problem), C.POINTER(_abi.Response), C.c_int32, C.c_int32,
                                       C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, _F64P, _U64P, C.c_char_p,
                                       C.c_size_t]),
    "ref_brute_force": (C.c_int, [_U64P, C.c_uint64, C.c_uint64, C.POINTER(C.c_int8), C.c_int32, C.c_double,
                                  C.c_int32, C.c_uint64, C.c_uint64, C.c_int32, C.POINTER(_U32P), C.POINTER(_F64P),
                                  _U64P, _U64P, C.POINTER(_U64P), C.c_char_p, C.c_size_t]),
}


class CheckerError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _load(path, sigs):
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `make -C oracle` (or __graft_entry__.build())")
    return _abi.bind(C.CDLL(path), sigs)


_cache = {}


def oracle_lib():
    if "o" not in _cache:
        _cache["o"] = _load(ORACLE_SO, _ORACLE_SIGS)
    return _cache["o"]


def ref_lib():
    if "r" not in _cache:
        _cache["r"] = _load(REF_SO, _REF_SIGS)
    return _cache["r"]


def ref_synth_lib():
    """The synthetic generators (csrc/synth.cpp) as linked into the checker
    library, bound with libxyzb_synth.so's signatures."""
    from paper_1610_05108_b200._lib import SYNTH_SIGNATURES
    if "rs" not in _cache:
        _cache["rs"] = _abi.bind(ref_lib(), SYNTH_SIGNATURES)
    return _cache["rs"]


def ref_available():
    return os.path.exists(REF_SO)


def _check(code, err):
    if code != 0:
        raise CheckerError(code, err.value.decode(errors="replace"))


def _search(lib, fn, free, x, y, cfg: SearchConfig):
    if isinstance(x, RealMatrix):
        x = x.as_float64()  # the reference takes doubles (double(x) of fp32 values)
    prob = make_problem(x)
    resp, keep = make_response(y)
    params = cfg.to_params()
    res = _abi.Result()
    err = _abi.errbuf()
    code = getattr(lib, fn)(C.byref(prob), C.byref(resp), C.byref(params), C.byref(res), err, _abi.ERRBUF)
    _check(code, err)
    try:
        return report_from_result(res)
    finally:
        getattr(lib, free)(C.byref(res))


def oracle_search(x, y, cfg):
    return _search(oracle_lib(), "oracle_search", "oracle_result_free", x, y, cfg)


def ref_search(x, y, cfg):
    return _search(ref_lib(), "ref_search", "ref_result_free", x, y, cfg)


def _u64p(a):
    return a.ctypes.data_as(_U64P)


def oracle_draws(n, m, l, negatives, seed, y=None):
    lib = oracle_lib()
    out = np.zeros(((2 if negatives else 1), l, m), np.uint32)
    err = _abi.errbuf()
    yy = None if y is None else np.ascontiguousarray(y, np.float64)
    _check(lib.oracle_draws(n, m, l, int(negatives), seed, None if yy is None else yy.ctypes.data_as(_F64P),
                            out.ctypes.data_as(_U32P), err, _abi.ERRBUF), err)
    return out


def oracle_project_keys(x: PackedMatrix, draws: np.ndarray):
    lib = oracle_lib()
    draws = np.ascontiguousarray(draws, np.uint32).reshape(-1, draws.shape[-1])
    keys = np.zeros((draws.shape[0], x.n_cols), np.uint64)
    err = _abi.errbuf()
    _check(lib.oracle_project_keys(_u64p(x.words), x.n_rows, x.n_cols, draws.ctypes.data_as(_U32P), draws.shape[0],
                                   draws.shape[1], _u64p(keys), err, _abi.ERRBUF), err)
    return keys


def _pairs(lib, fn, free, xk, zk):
    xk = np.ascontiguousarray(xk, np.uint64)
    zk = np.ascontiguousarray(zk, np.uint64)
    ptr = _U32P()
    npairs = C.c_uint64()
    total = C.c_uint64()
    err = _abi.errbuf()
    _check(getattr(lib, fn)(_u64p(xk), _u64p(zk), len(xk), C.byref(ptr), C.byref(npairs), C.byref(total), err,
                            _abi.ERRBUF), err)
    try:
        arr = np.ctypeslib.as_array(ptr, shape=(2 * npairs.value,)).copy().reshape(-1, 2) if npairs.value else \
            np.zeros((0, 2), np.uint32)
    finally:
        getattr(lib, free)(ptr)
    return arr, total.value


def oracle_equal_pairs(xk, zk):
    return _pairs(oracle_lib(), "oracle_equal_pairs", "oracle_free", xk, zk)


def ref_equal_pairs(xk, zk):
    return _pairs(ref_lib(), "ref_equal_pairs", "ref_free", xk, zk)


def _strengths(lib, fn, x, y, mode, transform, pairs):
    if isinstance(x, RealMatrix):
        x = x.as_float64()
    prob = make_problem(x)
    resp, keep = make_response(y)
    pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
    out = np.zeros(len(pairs), np.float64)
    err = _abi.errbuf()
    _check(getattr(lib, fn)(C.byref(prob), C.byref(resp), mode, transform, pairs.ctypes.data_as(_U32P), len(pairs),
                            out.ctypes.data_as(_F64P), err, _abi.ERRBUF), err)
    return out


def oracle_pair_strengths(x, y, mode, transform, pairs):
    return _strengths(oracle_lib(), "oracle_pair_strengths", x, y, mode, transform, pairs)


def ref_pair_strengths(x, y, mode, transform, pairs):
    return _strengths(ref_lib(), "ref_pair_strengths", x, y, mode, transform, pairs)


def ref_draw_subsample(n, m, seed, stream, y=None):
    lib = ref_lib()
    out = np.zeros(m, np.uint64)
    err = _abi.errbuf()
    yy = None if y is None else np.ascontiguousarray(y, np.float64)
    _check(lib.ref_draw_subsample(n, m, seed, stream, None if yy is None else yy.ctypes.data_as(_F64P), _u64p(out),
                                  err, _abi.ERRBUF), err)
    return out


def ref_project_keys(x: PackedMatrix, draw):
    lib = ref_lib()
    d = np.ascontiguousarray(draw, np.uint64)
    keys = np.zeros(x.n_cols, np.uint64)
    err = _abi.errbuf()
    _check(lib.ref_project_keys(_u64p(x.words), x.n_rows, x.n_cols, _u64p(d), len(d), _u64p(keys), err, _abi.ERRBUF),
           err)
    return keys


def ref_rademacher(n, p, seed, stream):
    lib = ref_lib()
    x = PackedMatrix(n, p)
    err = _abi.errbuf()
    _check(lib.ref_rademacher_matrix(n, p, seed, stream, _u64p(x.words), err, _abi.ERRBUF), err)
    return x


def ref_planted(n, p, j, k, gamma, seed, stream=0x5e17):
    lib = ref_lib()
    x = PackedMatrix(n, p)
    y = np.zeros(n, np.int8)
    err = _abi.errbuf()
    _check(lib.ref_planted_instance(n, p, j, k, gamma, seed, stream, _u64p(x.words),
                                    y.ctypes.data_as(C.POINTER(C.c_int8)), err, _abi.ERRBUF), err)
    return x, y


def ref_gaussian(n, p, seed, stream):
    lib = ref_lib()
    out = np.zeros((p, n), np.float64)
    err = _abi.errbuf()
    _check(lib.ref_gaussian_matrix(n, p, seed, stream, out.ctypes.data_as(_F64P), err, _abi.ERRBUF), err)
    return RealMatrix(out)


def ref_uniform(n, p, seed, stream):
    lib = ref_lib()
    out = np.zeros((p, n), np.float64)
    err = _abi.errbuf()
    _check(lib.ref_uniform_matrix(n, p, seed, stream, out.ctypes.data_as(_F64P), err, _abi.ERRBUF), err)
    return RealMatrix(out)


def ref_rescale_rows(x: RealMatrix, y):
    lib = ref_lib()
    xo = np.zeros_like(x.values)
    yy = np.ascontiguousarray(y, np.float64)
    yo = np.zeros_like(yy)
    err = _abi.errbuf()
    _check(lib.ref_rescale_rows(x.values.ctypes.data_as(_F64P), x.n_rows, x.n_cols, yy.ctypes.data_as(_F64P),
                                xo.ctypes.data_as(_F64P), yo.ctypes.data_as(_F64P), err, _abi.ERRBUF), err)
    return RealMatrix(xo), yo


def ref_brute_force_topk(x: PackedMatrix, y, k):
    lib = ref_lib()
    yy = np.ascontiguousarray(y, np.int8)
    jk = np.zeros((k, 2), np.uint32)
    s = np.zeros(k, np.float64)
    cnt = C.c_uint64()
    err = _abi.errbuf()
    _check(lib.ref_brute_force_topk(_u64p(x.words), x.n_rows, x.n_cols, yy.ctypes.data_as(C.POINTER(C.c_int8)), k,
                                    jk.ctypes.data_as(_U32P), s.ctypes.data_as(_F64P), C.byref(cnt), err,
                                    _abi.ERRBUF), err)
    return jk[: cnt.value], s[: cnt.value]


def same_hits(a, b, strength_tol=0.0):
    """Bit-exact (strength_tol=0) or tolerant comparison of two hit lists."""
    if len(a.hits) != len(b.hits):
        return False, f"hit count {len(a.hits)} != {len(b.hits)}"
    for i, (h, g) in enumerate(zip(a.hits, b.hits)):
        if (h.j, h.k, h.found_at_repetition, h.sign) != (g.j, g.k, g.found_at_repetition, g.sign):
            return False, f"hit {i}: {h} != {g}"
        if strength_tol == 0.0:
            if h.strength != g.strength:
                return False, f"hit {i} strength {h.strength!r} != {g.strength!r}"
        elif abs(h.strength - g.strength) > strength_tol * max(abs(g.strength), 1e-300):
            return False, f"hit {i} strength {h.strength!r} vs {g.strength!r} beyond {strength_tol}"
    return True, ""


# ---- the drop-in build: reference core with search.cpp replaced by the GPU shim ----

# the test harness over the drop-in (it pulls build/dropin/libxyz_core_gpu.so in)
DROPIN_SO = os.path.join(ROOT, "build", "dropin", "libxyz_core_gpu_harness.so")


class LassoOut(C.Structure):
    _fields_ = [("n_fits", C.c_uint64), ("lambda_", C.POINTER(C.c_double)), ("main_off", _U64P),
                ("main_idx", _U32P), ("main_val", _F64P), ("pair_off", _U64P), ("pair_j", _U32P),
                ("pair_k", _U32P), ("pair_val", _F64P), ("kkt_residual_max", _F64P),
                ("certified", C.POINTER(C.c_uint8)), ("degenerate", C.POINTER(C.c_uint8)),
                ("active_set_iterations", _U64P), ("cd_cycles", _U64P), ("wall_s", C.c_double)]


_LASSO_SIGS = {
    "ref_lasso_path": (C.c_int, [_F64P, C.c_uint64, C.c_uint64, _F64P, C.c_uint64, C.c_double, C.c_uint64,
                                 C.c_uint64, C.c_uint64, C.c_uint32, C.c_int32, C.POINTER(LassoOut), C.c_char_p,
                                 C.c_size_t]),
    "ref_lasso_free": (None, [C.POINTER(LassoOut)]),
    "ref_kkt_check_interactions": (C.c_int, [_F64P, C.c_uint64, C.c_uint64, _F64P, C.c_double, C.c_uint64, C.c_uint64,
                                             C.c_uint64, C.c_uint64, C.c_uint32, C.POINTER(_U32P),
                                             C.POINTER(C.c_uint64), C.c_char_p, C.c_size_t]),
}


def dropin_available():
    return os.path.exists(DROPIN_SO)


def dropin_lib():
    if "d" not in _cache:
        _cache["d"] = _load(DROPIN_SO, {**_REF_SIGS, **_LASSO_SIGS})
    return _cache["d"]


def ref_lasso_lib():
    if "rl" not in _cache:
        _cache["rl"] = _abi.bind(ref_lib(), _LASSO_SIGS)
    return _cache["rl"]


def dropin_search(x, y, cfg):
    return _search(dropin_lib(), "ref_search", "ref_result_free", x, y, cfg)


def lasso_path(lib, x: RealMatrix, y, grid_size=20, grid_ratio=0.05, kkt_l=0, kkt_max_candidates=0, seed=7,
               threads=1, certify=True):
    """lasso_path through a harness library; returns (fits, wall_s). Each fit:
    dict(lambda, beta {j: v}, theta {(j, k): v}, kkt, certified, degenerate)."""
    out = LassoOut()
    err = _abi.errbuf()
    yy = np.ascontiguousarray(y, np.float64)
    _check(lib.ref_lasso_path(x.values.ctypes.data_as(_F64P), x.n_rows, x.n_cols, yy.ctypes.data_as(_F64P),
                              grid_size, grid_ratio, kkt_l, kkt_max_candidates, seed, threads, int(certify),
                              C.byref(out), err, _abi.ERRBUF), err)
    fits = []
    try:
        for t in range(out.n_fits):
            beta = {int(out.main_idx[i]): float(out.main_val[i]) for i in range(out.main_off[t], out.main_off[t + 1])}
            theta = {(int(out.pair_j[i]), int(out.pair_k[i])): float(out.pair_val[i])
                     for i in range(out.pair_off[t], out.pair_off[t + 1])}
            fits.append(dict(lam=float(out.lambda_[t]), beta=beta, theta=theta, kkt=float(out.kkt_residual_max[t]),
                             certified=bool(out.certified[t]), degenerate=bool(out.degenerate[t]),
                             iterations=int(out.active_set_iterations[t])))
        return fits, out.wall_s
    finally:
        lib.ref_lasso_free(C.byref(out))


def kkt_check_interactions(lib, x: RealMatrix, residual, lam, kkt_l=0, kkt_max_candidates=0, seed=7, stream=1,
                           threads=1):
    """kkt_check_interactions through a harness library: sorted (j, k) list."""
    pj = _U32P()
    cnt = C.c_uint64(0)
    err = _abi.errbuf()
    r = np.ascontiguousarray(residual, np.float64)
    _check(lib.ref_kkt_check_interactions(x.values.ctypes.data_as(_F64P), x.n_rows, x.n_cols, r.ctypes.data_as(_F64P),
                                          lam, kkt_l, kkt_max_candidates, seed, stream, threads, C.byref(pj),
                                          C.byref(cnt), err, _abi.ERRBUF), err)
    try:
        return [(int(pj[2 * t]), int(pj[2 * t + 1])) for t in range(cnt.value)]
    finally:
        ref_lib().ref_free(pj)


def ref_write_dataset(path, x):
    lib = ref_lib()
    err = _abi.errbuf()
    if isinstance(x, PackedMatrix):
        _check(lib.ref_write_dataset(str(path).encode(), 0, _u64p(x.words), None, x.n_rows, x.n_cols, err, _abi.ERRBUF),
               err)
    else:
        _check(lib.ref_write_dataset(str(path).encode(), 1, None, x.values.ctypes.data_as(_F64P), x.n_rows, x.n_cols,
                                     err, _abi.ERRBUF), err)


def ref_read_dataset(path):
    """(kind, n, p) or raises CheckerError with the reference's message."""
    lib = ref_lib()
    kind, n, p = C.c_int32(), C.c_uint64(), C.c_uint64()
    err = _abi.errbuf()
    _check(lib.ref_read_dataset(str(path).encode(), C.byref(kind), C.byref(n), C.byref(p), err, _abi.ERRBUF), err)
    return kind.value, n.value, p.value


def ref_brute_force(x: PackedMatrix, y, gamma=None, top_k=None, histogram_bins=0, force=False):
    """oracle::brute_force_search of the reference: ([(j, k, s)], pairs_scanned, [hist]);
    the continuous-response overload when y is not int8."""
    lib = ref_lib()
    weighted = np.asarray(y).dtype != np.int8
    yy = np.ascontiguousarray(y, np.float64 if weighted else np.int8)
    jk, s, h = _U32P(), _F64P(), _U64P()
    n, scanned = C.c_uint64(), C.c_uint64()
    err = _abi.errbuf()
    fn = lib.ref_brute_force_weighted if weighted else lib.ref_brute_force
    code = fn(_u64p(x.words), x.n_rows, x.n_cols, yy.ctypes.data_as(_F64P if weighted else C.POINTER(C.c_int8)),
                               int(gamma is not None), float(gamma or 0.0), int(top_k is not None), int(top_k or 0),
                               int(histogram_bins), int(force), C.byref(jk), C.byref(s), C.byref(n),
                               C.byref(scanned), C.byref(h), err, _abi.ERRBUF)
    try:
        _check(code, err)
        pairs = [(jk[2 * i], jk[2 * i + 1], s[i]) for i in range(n.value)]
        hist = [h[i] for i in range(histogram_bins)]
    finally:
        for ptr in (jk, s, h):
            if ptr:
                lib.ref_free(ptr)
    return pairs, scanned.value, hist


# ---- top-K over all verified candidates ----

def topk_a10(hits, k):
    """A.10: the hit list stably sorted by (strength desc, min(j,k) asc,
    max(j,k) asc, sign desc) — oracle.cpp:45-56 extended with the sign —
    first k entries."""
    order = sorted(range(len(hits)), key=lambda i: (-hits[i].strength, min(hits[i].j, hits[i].k),
                                                    max(hits[i].j, hits[i].k), -hits[i].sign))
    return [hits[i] for i in order[:k]]


def ref_topk_candidates(x, y, cfg, k, gamma_start=0.6, step=0.01, threads=None):
    """A.10's gamma-lowering procedure on the unmodified reference: lower gamma
    on a grid (gamma_start, gamma_start - step, ...) until the reference's hit
    list holds >= k entries, then rank it. Returns (gamma_used, report, top-k hits)."""
    from dataclasses import replace
    g = gamma_start
    while True:
        rep = ref_search(x, y, replace(cfg, gamma=g, top_k=0, top_k_mode="hits",
                                       threads=threads or os.cpu_count() or 1))
        if len(rep.hits) >= k or g <= step:
            return g, rep, topk_a10(rep.hits, k)
        g = round(g - step, 12)


def hit_tuples(hits):
    return [(h.j, h.k, h.strength, h.found_at_repetition, h.sign) for h in hits]


def sample_strengths(lib, x, y, mode, transform, n_samples, seed=7, stream=0xdead, gamma=0.6):
    """xyz::sample_strengths + optimal_m through a harness library (the
    reference core, or the drop-in where they run on the GPU):
    (strengths, optimal M)."""
    if isinstance(x, RealMatrix):
        x = x.as_float64()
    prob = make_problem(x)
    resp, keep = make_response(y)
    out = np.zeros(n_samples, np.float64)
    m = C.c_uint64()
    err = _abi.errbuf()
    _check(lib.ref_sample_strengths(C.byref(prob), C.byref(resp), mode, transform, n_samples, seed, stream, gamma,
                                    out.ctypes.data_as(_F64P), C.byref(m), err, _abi.ERRBUF), err)
    return out, m.value
