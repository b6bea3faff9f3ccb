"""Host-side data layouts of the reference, as numpy views.

PackedMatrix mirrors proj/core/include/xyz/packed_matrix.hpp:10-57: column-major
uint64 words, W = ceil(n/64) per column, bit i%64 of word i/64 set iff
X_ij = +1, padding bits zero. RealMatrix mirrors real_matrix.hpp:13-33
(column-major doubles).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi


class PackedMatrix:
    def __init__(self, n_rows: int, n_cols: int, words: np.ndarray | None = None):
        if n_rows == 0 or n_cols == 0:
            raise ValueError("PackedMatrix: n_rows and n_cols must be >= 1")
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.words_per_col = (self.n_rows + 63) // 64
        if words is None:
            words = np.zeros((self.n_cols, self.words_per_col), np.uint64)
        words = np.ascontiguousarray(words, dtype=np.uint64).reshape(self.n_cols, self.words_per_col)
        self.words = words

    @staticmethod
    def from_signs(signs: np.ndarray) -> "PackedMatrix":
        """signs: int array (n, p) of +-1 (row i, column j)."""
        signs = np.asarray(signs)
        n, p = signs.shape
        bits = (signs > 0).astype(np.uint8).T  # (p, n)
        W = (n + 63) // 64
        padded = np.zeros((p, W * 64), np.uint8)
        padded[:, :n] = bits
        packed = np.packbits(padded.reshape(p, W, 64), axis=2, bitorder="little")  # (p, W, 8)
        return PackedMatrix(n, p, packed.view(np.uint64).reshape(p, W))

    def to_signs(self) -> np.ndarray:
        bits = np.unpackbits(self.words.view(np.uint8).reshape(self.n_cols, -1), axis=1, bitorder="little")
        return (bits[:, : self.n_rows].T.astype(np.int8) * 2 - 1)

    def get(self, i: int, j: int) -> int:
        return 1 if (int(self.words[j, i >> 6]) >> (i & 63)) & 1 else -1

    @property
    def last_word_mask(self) -> int:
        t = self.n_rows & 63
        return (1 << 64) - 1 if t == 0 else (1 << t) - 1

    def padding_clear(self) -> bool:
        return bool(np.all((self.words[:, -1] & np.uint64(~self.last_word_mask & ((1 << 64) - 1))) == 0))

    def column_words(self, j: int) -> np.ndarray:
        return self.words[j]


def pack_signs(y: np.ndarray) -> np.ndarray:
    """pack_signs (packed_matrix.cpp:29-35): +1 -> bit 1, padding 0."""
    y = np.asarray(y)
    n = y.shape[0]
    W = (n + 63) // 64
    bits = np.zeros(W * 64, np.uint8)
    bits[:n] = y > 0
    return np.packbits(bits.reshape(W, 64), axis=1, bitorder="little").view(np.uint64).reshape(W)


class RealMatrix:
    """Column-major doubles: values[j, i] = X_ij. Engine extension:
    dtype=np.float32 keeps float values (uploaded as x_real32, half the bytes;
    every comparison sees double(x), as a RealMatrix built from them)."""

    def __init__(self, values_colmajor: np.ndarray, dtype=np.float64):
        if np.dtype(dtype) not in (np.dtype(np.float64), np.dtype(np.float32)):
            raise ValueError("RealMatrix: dtype must be float64 or float32")
        v = np.ascontiguousarray(values_colmajor, dtype=dtype)
        if v.ndim != 2 or v.size == 0:
            raise ValueError("RealMatrix: need a non-empty (p, n) array")
        self.values = v
        self.n_cols, self.n_rows = v.shape

    @staticmethod
    def from_rows(x_rows: np.ndarray) -> "RealMatrix":
        """x_rows: (n, p) array, row i column j."""
        return RealMatrix(np.asarray(x_rows, np.float64).T)

    def __call__(self, i: int, j: int) -> float:
        return float(self.values[j, i])

    def column(self, j: int) -> np.ndarray:
        return self.values[j]

    def as_float64(self) -> "RealMatrix":
        return self if self.values.dtype == np.float64 else RealMatrix(self.values.astype(np.float64))


def make_problem(x, device: int = 0, devices=None):
    """Build an xyzb_problem pointing into x's buffer (x must outlive it).
    devices: replicate X on these devices (the search shards its runs over
    them); the returned problem keeps the device array alive."""
    prob = _abi.Problem()
    prob.device = device
    if isinstance(x, PackedMatrix):
        prob.n_rows, prob.n_cols = x.n_rows, x.n_cols
        prob.x_words = x.words.ctypes.data_as(C.POINTER(C.c_uint64))
    elif isinstance(x, RealMatrix):
        prob.n_rows, prob.n_cols = x.n_rows, x.n_cols
        if x.values.dtype == np.float32:
            prob.x_real32 = x.values.ctypes.data_as(C.POINTER(C.c_float))
        else:
            prob.x_real = x.values.ctypes.data_as(C.POINTER(C.c_double))
    else:
        raise TypeError("x must be a PackedMatrix or RealMatrix")
    if devices:
        arr = (C.c_int32 * len(devices))(*[int(d) for d in devices])
        prob.devices = C.cast(arr, C.POINTER(C.c_int32))
        prob.n_devices = len(devices)
        prob._keep = arr
    return prob


def make_response(y):
    """Build an xyzb_response; returns (response, keepalive array)."""
    resp = _abi.Response()
    y = np.asarray(y)
    if y.dtype == np.int8:
        arr = np.ascontiguousarray(y)
        resp.y_sign = arr.ctypes.data_as(C.POINTER(C.c_int8))
    else:
        arr = np.ascontiguousarray(y, dtype=np.float64)
        resp.y_real = arr.ctypes.data_as(C.POINTER(C.c_double))
    return resp, arr
