"""Multi-rank host logic on CPU (gloo, world size 2): run-shard bounds, result
serialisation, the variable-size all-gather, and the merge rule the device
merge implements (first occurrence of (min, max, sign) by order key, then
order-key order). The GPU test at the end runs the same world-size-2 gloo
exchange around real shard searches and the device merge (xyzb_merge_results)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

from paper_1610_05108_b200 import _abi, parallel
from paper_1610_05108_b200.report import SearchConfig


def test_shard_bounds_partition_the_repetitions():
    for L in (1, 2, 7, 100, 101):
        for W in (1, 2, 3, 4, 8):
            got = [parallel.shard_bounds(L, r, W) for r in range(W)]
            assert got[0][0] == 1 and got[-1][1] == L + 1
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            assert max(e - b for b, e in got) - min(e - b for b, e in got) <= 1


def test_shard_config_keeps_the_estimate_on_rank0_only():
    cfg = SearchConfig(l=10, estimate_complexity=True)
    assert parallel.shard_config(cfg, 0, 2).estimate_complexity
    assert not parallel.shard_config(cfg, 1, 2).estimate_complexity
    assert (parallel.shard_config(cfg, 1, 2).rep_begin, parallel.shard_config(cfg, 1, 2).rep_end) == (6, 11)


def make_result(hits, orders, **counters):
    """An ABI result pointing into numpy storage (kept alive on the object)."""
    r = _abi.Result()
    arr = np.zeros(len(hits), parallel._HIT_DT)
    for i, h in enumerate(hits):
        arr[i] = h
    order = np.array(orders, np.uint64)
    r.n_hits = len(hits)
    r.hits = arr.ctypes.data_as(C.POINTER(_abi.Hit)) if len(hits) else None
    r.order_keys = order.ctypes.data_as(C.POINTER(C.c_uint64)) if len(hits) else None
    for k, v in counters.items():
        setattr(r, k, v)
    r._keep = (arr, order)
    return r


def reference_merge(parts):
    """Appendix A.8 on gathered shard lists: keep the smallest order key per
    (min, max, sign), emit in order-key order."""
    best = {}
    for p in parts:
        a = p.hit_array()
        for h, o in zip(a, p.order):
            key = (min(h["j"], h["k"]), max(h["j"], h["k"]), int(h["sign"]))
            if key not in best or o < best[key][0]:
                best[key] = (int(o), (int(h["j"]), int(h["k"]), float(h["strength"]), int(h["rep"]), int(h["sign"])))
    return [v[1] for v in sorted(best.values())]


def test_pack_roundtrip():
    r = make_result([(3, 9, 0.75, 2, 1), (1, 4, 0.6, 5, -1)], [17, 99], repetitions_run=4,
                    candidates_enumerated=123, verified_pairs=55, estimated_c=1.5)
    part = parallel.PackedPart(parallel.pack_result(r))
    assert part.result.n_hits == 2
    assert part.result.repetitions_run == 4 and part.result.candidates_enumerated == 123
    assert part.result.verified_pairs == 55 and part.result.estimated_c == 1.5
    assert part.order.tolist() == [17, 99]
    assert part.hit_array()["j"].tolist() == [3, 1] and part.hit_array()["sign"].tolist() == [1, -1]
    empty = parallel.PackedPart(parallel.pack_result(make_result([], [])))
    assert empty.result.n_hits == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank-local, already deduplicated shard lists (rank 1 re-finds (3, 9, +1) later)
    if rank == 0:
        r = make_result([(3, 9, 0.75, 1, 1), (2, 8, 0.7, 2, 1)], [10, 25], repetitions_run=2,
                        candidates_enumerated=40)
    else:
        r = make_result([(9, 3, 0.75, 4, 1), (5, 6, 0.8, 3, 1), (2, 8, 0.3, 1, -1)], [70, 45, 205],
                        repetitions_run=2, candidates_enumerated=60)
    # ragged and all-empty byte buffers survive the padded exchange
    raw = parallel.all_gather_bytes(np.arange(3 + 5 * rank, dtype=np.uint8))
    assert [b.tolist() for b in raw] == [list(range(3)), list(range(8))]
    assert [b.size for b in parallel.all_gather_bytes(np.zeros(0, np.uint8))] == [0, 0]
    gathered = parallel.all_gather_bytes(parallel.pack_result(r))
    parts = [parallel.PackedPart(b) for b in gathered]
    merged = reference_merge(parts)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"),
            np.array([merged, sum(p.result.candidates_enumerated for p in parts)], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gather_and_merge_on_gloo(tmp_path):
    import torch.multiprocessing as mp
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npy", allow_pickle=True)
    r1 = np.load(tmp_path / "rank1.npy", allow_pickle=True)
    assert r0[0] == r1[0]  # every rank merges to the same report
    assert r0[0] == [(3, 9, 0.75, 1, 1), (2, 8, 0.7, 2, 1), (5, 6, 0.8, 3, 1), (2, 8, 0.3, 1, -1)]
    assert r0[1] == 100


def _engine_worker(rank, world, port, out_dir, topk_mode):
    """One rank of a sharded search on the GPU: its repetition shard, the gloo
    all-gather of the serialised shard results, and the device merge through
    xyzb_merge_results (parallel.sharded_search — bench.py's N>1 path)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    import paper_1610_05108_b200 as xb
    from tests import checkers as ck
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x = ck.ref_rademacher(900, 1500, 31, 2)
    y = np.where(np.random.default_rng(4).random(900) < 0.5, 1, -1).astype(np.int8)
    cfg = SearchConfig(m=8, l=12, gamma=0.56, seed=7, top_k=40, top_k_mode=topk_mode, threads=1)
    ds = xb.Dataset(x, device=0)
    rep = parallel.sharded_search(ds, y, cfg, rank, world)
    import pickle
    with open(os.path.join(out_dir, f"engine{rank}.pkl"), "wb") as f:
        pickle.dump([ck.hit_tuples(rep.hits), rep.top_k, rep.candidates_enumerated, rep.repetitions_run,
                     rep.gamma_effective], f)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("topk_mode", ["hits", "candidates"])
def test_two_rank_engine_search_gloo_merges_on_the_device(tmp_path, topk_mode):
    """World size 2 on gloo with both ranks on the test box's GPU (independent
    searches, no kernel waits on another rank): the merged report of every
    rank equals the unsharded search."""
    import torch.multiprocessing as mp
    import paper_1610_05108_b200 as xb
    from tests import checkers as ck
    port = _free_port()
    mp.spawn(_engine_worker, args=(2, port, str(tmp_path), topk_mode), nprocs=2, join=True)
    x = ck.ref_rademacher(900, 1500, 31, 2)
    y = np.where(np.random.default_rng(4).random(900) < 0.5, 1, -1).astype(np.int8)
    cfg = SearchConfig(m=8, l=12, gamma=0.56, seed=7, top_k=40, top_k_mode=topk_mode, threads=1)
    whole = xb.Dataset(x).search(y, cfg)
    import pickle
    for r in (0, 1):
        with open(tmp_path / f"engine{r}.pkl", "rb") as f:
            got = pickle.load(f)
        assert got[0] == ck.hit_tuples(whole.hits)
        assert got[1] == whole.top_k
        assert (got[2], got[3], got[4]) == (whole.candidates_enumerated, whole.repetitions_run,
                                            whole.gamma_effective)
