"""B200-native xyz interaction search (arXiv 1610.05108 hot path).

The product is libxyzb.so (CUDA sm_100a + host C++, C ABI in include/xyzb.h);
this package is its Python host mirror, named after the reference's C++ API
(proj/core/include/xyz/search.hpp, packed_matrix.hpp, real_matrix.hpp).
"""
from ._lib import CudaError, DataError, EngineError, GuardError, SolverError, XyzError
from .engine import (Dataset, OracleResult, ScoredPair, brute_force_search, dataset_for, device_count, equal_pairs,
                     xyz_search)
from .matrix import PackedMatrix, RealMatrix, pack_signs
from .report import (BINARY, CONTINUOUS_XY, CONTINUOUS_Y, NONE, SIGN, UNBIASED, InteractionHit, SearchConfig,
                     SearchReport)

__all__ = [
    "xyz_search", "Dataset", "dataset_for", "device_count", "equal_pairs",
    "brute_force_search", "OracleResult", "ScoredPair",
    "PackedMatrix", "RealMatrix", "pack_signs",
    "SearchConfig", "SearchReport", "InteractionHit",
    "BINARY", "CONTINUOUS_Y", "CONTINUOUS_XY", "NONE", "SIGN", "UNBIASED",
    "XyzError", "DataError", "GuardError", "SolverError", "CudaError", "EngineError",
]
