"""Python host mirror of the reference's search entry points over libxyzb.so.

`xyz_search(x, y, config)` dispatches like the three C++ overloads
(proj/core/include/xyz/search.hpp:100-111):
  PackedMatrix + int8 +-1 vector  -> binary
  PackedMatrix + float vector     -> continuous-Y
  RealMatrix   + float vector     -> continuous-XY
and raises DataError where the reference throws xyz::data_error.

`Dataset` keeps X resident in HBM across calls (the ABI's dataset handle);
`xyz_search` caches one Dataset per X object.
"""
from __future__ import annotations

import ctypes as C
import weakref
from typing import NamedTuple, Optional, Sequence

import numpy as np

from . import _abi
from ._lib import DataError, load, raise_for
from .matrix import PackedMatrix, RealMatrix, make_problem, make_response
from .report import BINARY, CONTINUOUS_XY, CONTINUOUS_Y, SearchConfig, SearchReport, report_from_result


class Dataset:
    """X uploaded once to one GPU (xyzb_dataset_create), or replicated on
    several (`devices`: the search shards its runs over them and merges the
    shard results on devices[0] — SURVEY 8e)."""

    def __init__(self, x, device: int = 0, devices: Optional[Sequence[int]] = None):
        self._lib = load()
        self.x = x
        self.device = devices[0] if devices else device
        self.devices = list(devices) if devices else [device]
        self.binary = isinstance(x, PackedMatrix)
        self.n_rows, self.n_cols = x.n_rows, x.n_cols
        prob = make_problem(x, device, devices)
        h = C.c_void_p()
        err = _abi.errbuf()
        raise_for(self._lib.xyzb_dataset_create(C.byref(prob), C.byref(h), err, _abi.ERRBUF), err)
        self._h = h
        self._fin = weakref.finalize(self, self._lib.xyzb_dataset_destroy, h)

    @classmethod
    def open(cls, path, device: int = 0) -> "Dataset":
        """X read straight from an XYZ1 file (read_dataset, dataset_io.cpp:91-129)
        into HBM; `x` is None (the matrix never lives on the host)."""
        self = cls.__new__(cls)
        self._lib = load()
        self.x = None
        self.device = device
        h = C.c_void_p()
        err = _abi.errbuf()
        raise_for(self._lib.xyzb_dataset_open(str(path).encode(), device, C.byref(h), err, _abi.ERRBUF), err)
        n, p, b = C.c_uint64(), C.c_uint64(), C.c_int32()
        self._lib.xyzb_dataset_shape(h, C.byref(n), C.byref(p), C.byref(b))
        self.n_rows, self.n_cols, self.binary = n.value, p.value, bool(b.value)
        self._h = h
        self._fin = weakref.finalize(self, self._lib.xyzb_dataset_destroy, h)
        return self

    @property
    def handle(self):
        return self._h

    def close(self):
        self._fin()

    def search(self, y, config: SearchConfig, draws: Optional[np.ndarray] = None) -> SearchReport:
        resp, keep = make_response(y)
        params = config.to_params()
        res = _abi.Result()
        err = _abi.errbuf()
        dptr = None
        if draws is not None:
            draws = np.ascontiguousarray(draws, np.uint32)
            dptr = draws.ctypes.data_as(C.POINTER(C.c_uint32))
        code = self._lib.xyzb_search(self._h, C.byref(resp), C.byref(params), dptr, C.byref(res), err, _abi.ERRBUF)
        try:
            raise_for(code, err)
            return report_from_result(res)
        finally:
            self._lib.xyzb_result_free(C.byref(res))

    def search_raw(self, y, config: SearchConfig) -> _abi.Result:
        """Search, returning the ABI result struct (caller frees with free_result)."""
        resp, keep = make_response(y)
        params = config.to_params()
        res = _abi.Result()
        err = _abi.errbuf()
        code = self._lib.xyzb_search(self._h, C.byref(resp), C.byref(params), None, C.byref(res), err, _abi.ERRBUF)
        if code != _abi.OK:
            self._lib.xyzb_result_free(C.byref(res))
        raise_for(code, err)
        return res

    def free_result(self, res: _abi.Result):
        self._lib.xyzb_result_free(C.byref(res))

    def project_keys(self, draws: np.ndarray) -> np.ndarray:
        """Keys of every column for each row of `draws` (n_draws, M)."""
        draws = np.ascontiguousarray(draws, np.uint32)
        if draws.ndim == 1:
            draws = draws[None, :]
        keys = np.zeros((draws.shape[0], self.n_cols), np.uint64)
        err = _abi.errbuf()
        raise_for(self._lib.xyzb_project_keys(self._h, draws.ctypes.data_as(C.POINTER(C.c_uint32)), draws.shape[0],
                                              draws.shape[1], keys.ctypes.data_as(C.POINTER(C.c_uint64)), err,
                                              _abi.ERRBUF), err)
        return keys

    def pair_strengths(self, y, config: SearchConfig, pairs) -> np.ndarray:
        resp, keep = make_response(y)
        params = config.to_params()
        pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        out = np.zeros(len(pairs), np.float64)
        err = _abi.errbuf()
        raise_for(self._lib.xyzb_pair_strengths(self._h, C.byref(resp), C.byref(params),
                                                pairs.ctypes.data_as(C.POINTER(C.c_uint32)), len(pairs),
                                                out.ctypes.data_as(C.POINTER(C.c_double)), err, _abi.ERRBUF), err)
        return out

    def pair_agreements(self, z: "Dataset", pairs) -> np.ndarray:
        """count_agreements(z_j, x_k) with this dataset as X (xyzb_pair_agreements)."""
        pairs = np.ascontiguousarray(pairs, np.uint32).reshape(-1, 2)
        out = np.zeros(len(pairs), np.uint64)
        err = _abi.errbuf()
        raise_for(self._lib.xyzb_pair_agreements(z.handle, self._h, pairs.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                 len(pairs), out.ctypes.data_as(C.POINTER(C.c_uint64)), err,
                                                 _abi.ERRBUF), err)
        return out

    def merge(self, parts: Sequence[_abi.Result], config: SearchConfig) -> SearchReport:
        arr = (_abi.Result * len(parts))(*parts)
        params = config.to_params()
        res = _abi.Result()
        err = _abi.errbuf()
        code = self._lib.xyzb_merge_results(self._h, arr, len(parts), C.byref(params), C.byref(res), err,
                                            _abi.ERRBUF)
        try:
            raise_for(code, err)
            return report_from_result(res)
        finally:
            self._lib.xyzb_result_free(C.byref(res))


_cache: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def dataset_for(x, device: int = 0) -> Dataset:
    ds = _cache.get(x)
    if ds is None or ds.device != device:
        ds = Dataset(x, device)
        _cache[x] = ds
    return ds


def xyz_search(x, y, config: SearchConfig, device: int = 0) -> SearchReport:
    """The three xyz::xyz_search overloads (search.cpp:325,367,415)."""
    y = np.asarray(y)
    if isinstance(x, PackedMatrix):
        if y.dtype == np.int8:
            if config.mode != BINARY:
                raise DataError("xyz_search: packed X with sign Y requires binary mode")
        elif config.mode != CONTINUOUS_Y:
            raise DataError("xyz_search: packed X with real Y requires continuous-Y mode")
    elif isinstance(x, RealMatrix):
        if config.mode != CONTINUOUS_XY:
            raise DataError("xyz_search: real X requires continuous-XY mode")
    else:
        raise TypeError("x must be a PackedMatrix or a RealMatrix")
    if y.shape[0] != x.n_rows:
        raise DataError("xyz_search: response length mismatch")
    return dataset_for(x, device).search(y, config)


def equal_pairs(x_keys, z_keys, device: int = 0):
    """equal_pairs (pair_search.cpp:26-55) on the GPU: candidate (j, k) pairs in
    filter order (key asc, j asc, k asc) and total_pairs."""
    lib = load()
    xk = np.ascontiguousarray(x_keys, np.uint64)
    zk = np.ascontiguousarray(z_keys, np.uint64)
    if xk.shape != zk.shape:
        raise DataError("equal_pairs: key vectors differ in length")
    ptr = C.POINTER(C.c_uint32)()
    npairs = C.c_uint64()
    total = C.c_uint64()
    err = _abi.errbuf()
    raise_for(lib.xyzb_equal_pairs(xk.ctypes.data_as(C.POINTER(C.c_uint64)), zk.ctypes.data_as(C.POINTER(C.c_uint64)),
                                   len(xk), device, C.byref(ptr), C.byref(npairs), C.byref(total), err, _abi.ERRBUF),
              err)
    try:
        if npairs.value:
            arr = np.ctypeslib.as_array(ptr, shape=(2 * npairs.value,)).copy().reshape(-1, 2)
        else:
            arr = np.zeros((0, 2), np.uint32)
    finally:
        lib.xyzb_free(ptr)
    return arr, total.value


def device_count() -> int:
    return int(load().xyzb_device_count())


class ScoredPair(NamedTuple):
    """oracle::ScoredPair (oracle.hpp:15-19)."""
    j: int
    k: int
    strength: float


class OracleResult(NamedTuple):
    """oracle::OracleResult (oracle.hpp:21-25)."""
    pairs: list
    pairs_scanned: int
    histogram: list


def brute_force_search(x, y, gamma: Optional[float] = None, top_k: Optional[int] = None, histogram_bins: int = 0,
                       force: bool = False, device: int = 0) -> OracleResult:
    """oracle::brute_force_search (oracle.hpp:36-41, oracle.cpp:84-100) on
    the GPU: exact strengths of all p(p-1)/2 pairs. `x` is a PackedMatrix or a
    binary Dataset; y the +-1 response (int8: tensor-core Gram product) or a
    real response (the weighted strength, bit-identical to the host's)."""
    ds = x if isinstance(x, Dataset) else dataset_for(x, device)
    weighted = np.asarray(y).dtype != np.int8  # the continuous-response overload (oracle.cpp:93-100)
    yy = np.ascontiguousarray(y, np.float64 if weighted else np.int8)
    if yy.shape[0] != ds.n_rows:
        raise DataError("brute_force_search: response length mismatch")
    lib = ds._lib
    pairs = C.POINTER(_abi.ScoredPair)()
    hist = C.POINTER(C.c_uint64)()
    npairs, scanned = C.c_uint64(), C.c_uint64()
    err = _abi.errbuf()
    fn = lib.xyzb_brute_force_weighted if weighted else lib.xyzb_brute_force
    yp = yy.ctypes.data_as(C.POINTER(C.c_double) if weighted else C.POINTER(C.c_int8))
    raise_for(fn(ds.handle, yp, int(gamma is not None), float(gamma) if gamma is not None else 0.0,
                 int(top_k is not None), int(top_k) if top_k is not None else 0, int(histogram_bins),
                 int(bool(force)), C.byref(pairs), C.byref(npairs), C.byref(scanned), C.byref(hist), err,
                 _abi.ERRBUF), err)
    try:
        out = [ScoredPair(pairs[i].j, pairs[i].k, pairs[i].strength) for i in range(npairs.value)]
        h = [int(hist[i]) for i in range(histogram_bins)] if histogram_bins and hist else []
    finally:
        lib.xyzb_free(pairs)
        lib.xyzb_free(hist)
    return OracleResult(out, scanned.value, h)
