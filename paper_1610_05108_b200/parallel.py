"""Run sharding across GPUs: one process per GPU, X replicated,
the 2L runs of a search split into contiguous repetition ranges per rank, one
all-gather of the per-rank deduplicated hit lists over NCCL (NVLink), and the
deterministic device merge (xyzb_merge_results) on every rank. The merged
report is identical for any world size (tests/test_gpu_parity.py,
tests/test_multirank.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import replace
from typing import List, Tuple

import numpy as np

from . import _abi
from .report import SearchConfig, SearchReport

_COUNTERS = ("repetitions_run", "candidates_checked", "candidates_enumerated", "aborted_repetitions",
             "runs_executed", "verified_pairs", "kernel_launches", "verify_launches", "devices_used", "attempts")
_FLOATS = ("wall_time_s", "estimated_c", "gamma0", "device_ms", "verify_kernel_ms", "gamma_effective")
_HIT_DT = np.dtype({"names": ["j", "k", "strength", "rep", "sign"], "formats": ["<u4", "<u4", "<f8", "<u4", "<i4"],
                    "offsets": [0, 4, 8, 16, 20], "itemsize": C.sizeof(_abi.Hit)})


def shard_bounds(l: int, rank: int, world: int) -> Tuple[int, int]:
    """1-based, end-exclusive repetition range of `rank` (balanced, contiguous)."""
    return 1 + (l * rank) // world, 1 + (l * (rank + 1)) // world


def shard_config(cfg: SearchConfig, rank: int, world: int) -> SearchConfig:
    b, e = shard_bounds(cfg.l, rank, world)
    # the complexity estimate is a per-search quantity: rank 0 computes it once
    return replace(cfg, rep_begin=b, rep_end=e, estimate_complexity=cfg.estimate_complexity and rank == 0)


def pack_result(res: _abi.Result) -> np.ndarray:
    """Serialise an ABI result (hits, order keys, counters) into bytes."""
    n = int(res.n_hits)
    head = np.zeros(4 + len(_COUNTERS) + len(_FLOATS) + 3 * _abi.NUM_STAGES, np.float64)
    ints = np.array([n] + [getattr(res, c) for c in _COUNTERS], np.uint64)
    flts = np.array([getattr(res, f) for f in _FLOATS], np.float64)
    st = np.concatenate([np.array(res.stage_ms[:], np.float64),
                         np.array(res.stage_bytes[:], np.uint64).view(np.float64),
                         np.array(res.stage_launches[:], np.uint64).view(np.float64)])
    head = np.concatenate([ints.view(np.float64), flts, st])
    hits = np.ctypeslib.as_array(C.cast(res.hits, C.POINTER(C.c_uint8)), shape=(n * _HIT_DT.itemsize,)) if n else \
        np.zeros(0, np.uint8)
    order = np.ctypeslib.as_array(res.order_keys, shape=(n,)).view(np.uint8) if n else np.zeros(0, np.uint8)
    return np.concatenate([np.array([len(head)], np.uint64).view(np.uint8), head.view(np.uint8), hits, order])


class PackedPart:
    """An unpacked result, exposed as an ABI struct for xyzb_merge_results."""

    def __init__(self, buf: np.ndarray):
        buf = np.ascontiguousarray(buf, np.uint8)
        nh = int(buf[:8].view(np.uint64)[0])
        head = buf[8:8 + 8 * nh].view(np.float64)
        off = 8 + 8 * nh
        ints = head[: 1 + len(_COUNTERS)].view(np.uint64)
        n = int(ints[0])
        flts = head[1 + len(_COUNTERS): 1 + len(_COUNTERS) + len(_FLOATS)]
        st = head[1 + len(_COUNTERS) + len(_FLOATS):]
        self.hits = buf[off: off + n * _HIT_DT.itemsize].copy()
        off += n * _HIT_DT.itemsize
        self.order = buf[off: off + 8 * n].copy().view(np.uint64)
        r = _abi.Result()
        r.n_hits = n
        if n:
            r.hits = self.hits.ctypes.data_as(C.POINTER(_abi.Hit))
            r.order_keys = self.order.ctypes.data_as(C.POINTER(C.c_uint64))
        for i, c in enumerate(_COUNTERS):
            setattr(r, c, int(ints[1 + i]))
        for i, f in enumerate(_FLOATS):
            setattr(r, f, float(flts[i]))
        S = _abi.NUM_STAGES
        for s in range(S):
            r.stage_ms[s] = float(st[s])
            r.stage_bytes[s] = int(st[S + s:S + s + 1].view(np.uint64)[0])
            r.stage_launches[s] = int(st[2 * S + s:2 * S + s + 1].view(np.uint64)[0])
        self.result = r

    def hit_array(self):
        return self.hits.view(_HIT_DT)


def all_gather_bytes(buf: np.ndarray, device=None) -> List[np.ndarray]:
    """All-gather variable-length byte buffers (sizes first, then a padded
    payload) with torch.distributed (NCCL on GPUs, gloo on CPU)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size()
    dev = device if device is not None else torch.device("cpu")
    size = torch.tensor([buf.size], dtype=torch.int64, device=dev)
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, size)
    m = max(1, int(max(int(s.item()) for s in sizes)))  # all-empty buffers still exchange one padded byte
    pad = np.zeros(m, np.uint8)
    pad[: buf.size] = buf
    t = torch.from_numpy(pad).to(dev)
    outs = [torch.zeros(m, dtype=torch.uint8, device=dev) for _ in range(world)]
    dist.all_gather(outs, t)
    return [o.cpu().numpy()[: int(s.item())] for o, s in zip(outs, sizes)]


def sharded_search(ds, y, cfg: SearchConfig, rank: int, world: int, device=None) -> SearchReport:
    """This rank's shard of the runs on its GPU, then gather + merge."""
    res = ds.search_raw(y, shard_config(cfg, rank, world))
    try:
        mine = pack_result(res)
    finally:
        ds.free_result(res)
    if world == 1:
        parts = [PackedPart(mine)]
    else:
        parts = [PackedPart(b) for b in all_gather_bytes(mine, device)]
    return ds.merge([p.result for p in parts], cfg)
