"""Python mirror of the reference's search-facing types.

`SearchConfig`, `SearchReport` and `InteractionHit` mirror
proj/core/include/xyz/search.hpp:18-56 and pair_search.hpp:29-35 field for
field (same names, same defaults, same meaning), so parity tests read like the
reference's own tests (proj/tests/test_search.cpp).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _abi

# SearchMode / BinarizeTransform (search.hpp:14-16)
BINARY, CONTINUOUS_Y, CONTINUOUS_XY = "binary", "continuous_y", "continuous_xy"
NONE, SIGN, UNBIASED = "none", "sign", "unbiased"
_MODES = {BINARY: _abi.MODE_BINARY, CONTINUOUS_Y: _abi.MODE_CONTINUOUS_Y, CONTINUOUS_XY: _abi.MODE_CONTINUOUS_XY}
_TRANSFORMS = {NONE: _abi.TRANSFORM_NONE, SIGN: _abi.TRANSFORM_SIGN, UNBIASED: _abi.TRANSFORM_UNBIASED}
# top_k_mode: "hits" = top-K of the hits (strength >= gamma); "candidates" = top-K over all verified
# candidates (gamma ignored; hits = the A.8 list at gamma_effective, the K-th strength)
TOPK_HITS, TOPK_CANDIDATES = "hits", "candidates"
_TOPK_MODES = {TOPK_HITS: _abi.TOPK_HITS, TOPK_CANDIDATES: _abi.TOPK_CANDIDATES}


@dataclass
class SearchConfig:
    """SearchConfig (search.hpp:18-33), defaults identical."""
    m: int = 8
    l: int = 1
    gamma: float = 0.9
    mode: str = BINARY
    transform: str = NONE
    search_negatives: bool = True
    seed: int = 0
    max_candidates_per_rep: int = 0
    stop_after_first_hit: bool = False
    estimate_complexity: bool = True
    threads: int = 0
    strength_sample_size: int = 0
    # engine extensions
    top_k: int = 0
    rep_begin: int = 0
    rep_end: int = 0
    top_k_mode: str = TOPK_HITS

    def to_params(self) -> _abi.Params:
        q = _abi.Params()
        q.m, q.l, q.gamma = self.m, self.l, self.gamma
        q.mode = _MODES[self.mode]
        q.transform = _TRANSFORMS[self.transform]
        q.search_negatives = int(self.search_negatives)
        q.stop_after_first_hit = int(self.stop_after_first_hit)
        q.estimate_complexity = int(self.estimate_complexity)
        q.threads = self.threads
        q.seed = self.seed & 0xFFFFFFFFFFFFFFFF
        q.max_candidates_per_rep = self.max_candidates_per_rep
        q.strength_sample_size = self.strength_sample_size
        q.top_k = self.top_k
        q.rep_begin, q.rep_end = self.rep_begin, self.rep_end
        q.top_k_mode = _TOPK_MODES[self.top_k_mode]
        return q


@dataclass
class InteractionHit:
    """InteractionHit (pair_search.hpp:29-35)."""
    j: int
    k: int
    strength: float
    found_at_repetition: int
    sign: int


@dataclass
class SearchReport:
    """SearchReport (search.hpp:45-56) plus engine telemetry."""
    hits: List[InteractionHit] = field(default_factory=list)
    repetitions_run: int = 0
    candidates_checked: int = 0
    candidates_enumerated: int = 0
    aborted_repetitions: int = 0
    wall_time_s: float = 0.0
    estimated_c: float = 0.0
    gamma0: float = 0.0
    m_used: int = 0
    l_used: int = 0
    top_k: List[int] = field(default_factory=list)
    order_keys: Optional[np.ndarray] = None
    runs_executed: int = 0
    verified_pairs: int = 0
    device_ms: float = 0.0
    stage_ms: dict = field(default_factory=dict)
    stage_bytes: dict = field(default_factory=dict)
    stage_launches: dict = field(default_factory=dict)
    kernel_launches: int = 0
    verify_kernel_ms: float = 0.0
    verify_launches: int = 0
    gamma_effective: float = 0.0
    devices_used: int = 0
    attempts: int = 1

    def hit_array(self) -> np.ndarray:
        """Hits as a structured array (j, k, strength, rep, sign)."""
        dt = np.dtype([("j", "<u4"), ("k", "<u4"), ("strength", "<f8"), ("rep", "<u4"), ("sign", "<i4")])
        a = np.zeros(len(self.hits), dt)
        for i, h in enumerate(self.hits):
            a[i] = (h.j, h.k, h.strength, h.found_at_repetition, h.sign)
        return a

    def top_hits(self) -> List[InteractionHit]:
        return [self.hits[i] for i in self.top_k]


def report_from_result(res: _abi.Result) -> SearchReport:
    n = int(res.n_hits)
    r = SearchReport()
    if n:
        raw = np.ctypeslib.as_array(C.cast(res.hits, C.POINTER(C.c_uint8)), shape=(n * C.sizeof(_abi.Hit),))
        dt = np.dtype({"names": ["j", "k", "strength", "rep", "sign"],
                       "formats": ["<u4", "<u4", "<f8", "<u4", "<i4"],
                       "offsets": [0, 4, 8, 16, 20], "itemsize": C.sizeof(_abi.Hit)})
        arr = raw.view(dt)
        r.hits = [InteractionHit(int(a["j"]), int(a["k"]), float(a["strength"]), int(a["rep"]), int(a["sign"]))
                  for a in arr]
        if res.order_keys:
            r.order_keys = np.ctypeslib.as_array(res.order_keys, shape=(n,)).copy()
    if res.n_top_k:
        r.top_k = [int(v) for v in np.ctypeslib.as_array(res.top_k, shape=(int(res.n_top_k),))]
    for name in ("repetitions_run", "candidates_checked", "candidates_enumerated", "aborted_repetitions",
                 "wall_time_s", "estimated_c", "gamma0", "m_used", "l_used", "runs_executed",
                 "verified_pairs", "device_ms", "kernel_launches", "verify_kernel_ms", "verify_launches",
                 "gamma_effective", "devices_used", "attempts"):
        setattr(r, name, getattr(res, name))
    r.stage_ms = {k: float(res.stage_ms[i]) for i, k in enumerate(_abi.STAGE_NAMES)}
    r.stage_bytes = {k: int(res.stage_bytes[i]) for i, k in enumerate(_abi.STAGE_NAMES)}
    r.stage_launches = {k: int(res.stage_launches[i]) for i, k in enumerate(_abi.STAGE_NAMES)}
    return r
