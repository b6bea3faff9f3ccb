"""Seeded synthetic inputs with BASELINE.json's config shapes (libxyzb_synth.so;
recipes in include/xyzb_synth.h). `lib`: another library exporting the same
generators (the reference arm uses the checker library oracle/_ref/libxyzref.so,
which links csrc/synth.cpp, so it loads none of the product-side libraries)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DataError, load_synth
from .matrix import PackedMatrix, RealMatrix

_U64P = C.POINTER(C.c_uint64)
_U32P = C.POINTER(C.c_uint32)
_F64P = C.POINTER(C.c_double)
_I8P = C.POINTER(C.c_int8)


def _chk(code):
    if code != 0:
        raise DataError(f"synthetic generator rejected its arguments (code {code})")


def toy(n=1000, p=2000, j=4, k=16, gamma=0.9, seed=1, lib=None):
    """Config 1: rademacher_matrix + plant_interaction on make_stream(seed, 0x5e17)."""
    x = PackedMatrix(n, p)
    y = np.zeros(n, np.int8)
    _chk((lib or load_synth()).xyzb_synth_toy(n, p, j, k, gamma, seed, x.words.ctypes.data_as(_U64P), y.ctypes.data_as(_I8P)))
    return x, y


def gwas(n=4000, p=100000, n_pairs=5, coef=1.5, seed=12345, lib=None):
    """Config 2: binarised Binomial(2, maf) genotypes, logistic Y with planted pairs."""
    x = PackedMatrix(n, p)
    y = np.zeros(n, np.int8)
    pairs = np.zeros((n_pairs, 2), np.uint32)
    _chk((lib or load_synth()).xyzb_synth_gwas(n, p, n_pairs, coef, seed, x.words.ctypes.data_as(_U64P),
                                      y.ctypes.data_as(_I8P), pairs.ctypes.data_as(_U32P)))
    return x, y, pairs


def gauss(n=2000, p=50000, n_pairs=10, theta=0.8, noise_sd=1.0, n_mains=0, beta=1.0, seed=3, lib=None):
    """Config 3 (and 5 with mains): standardised N(0,1) columns, planted products."""
    xv = np.zeros((p, n), np.float64)
    y = np.zeros(n, np.float64)
    pairs = np.zeros((n_pairs, 2), np.uint32)
    mains = np.zeros(max(n_mains, 1), np.uint32)
    _chk((lib or load_synth()).xyzb_synth_gauss(n, p, n_pairs, theta, noise_sd, n_mains, beta, seed,
                                       xv.ctypes.data_as(_F64P), y.ctypes.data_as(_F64P),
                                       pairs.ctypes.data_as(_U32P), mains.ctypes.data_as(_U32P)))
    return RealMatrix(xv), y, pairs, mains[:n_mains]


def ar1(n=10000, p=1000000, block=50, rho=0.3, n_pairs=20, flip=0.15, seed=99, lib=None):
    """Config 4: thresholded AR(1) Gaussian column blocks, sign-of-sum Y with flips."""
    x = PackedMatrix(n, p)
    y = np.zeros(n, np.int8)
    pairs = np.zeros((n_pairs, 2), np.uint32)
    _chk((lib or load_synth()).xyzb_synth_ar1(n, p, block, rho, n_pairs, flip, seed, x.words.ctypes.data_as(_U64P),
                                     y.ctypes.data_as(_I8P), pairs.ctypes.data_as(_U32P)))
    return x, y, pairs
