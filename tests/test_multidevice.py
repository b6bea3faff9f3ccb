"""Multi-device search behind the C ABI (SURVEY 8b device list, 8e): a
dataset replicated on several devices (xyzb_problem.devices) shards the
repetitions of each pass over them — one host thread and stream per device —
and merges the shard results on the first device. The report equals the
single-device search. On the one-GPU test box the "devices" are two or three
replicas on device 0: distinct datasets, streams and host threads running
concurrently, which is exactly the code path of distinct GPUs (the peer
copies become device-to-device copies)."""
from dataclasses import replace

import numpy as np
import pytest

from tests import checkers as ck

pytestmark = pytest.mark.gpu


def _xb():
    import paper_1610_05108_b200 as xb
    return xb


def _same(a, b, exact=True):
    assert ck.hit_tuples(a.hits) == ck.hit_tuples(b.hits)
    assert a.top_k == b.top_k
    for f in ("repetitions_run", "aborted_repetitions", "candidates_enumerated", "verified_pairs", "gamma0"):
        assert getattr(a, f) == getattr(b, f), f
    assert a.estimated_c == b.estimated_c
    assert a.gamma_effective == b.gamma_effective


@pytest.mark.parametrize("ndev", [2, 3])
@pytest.mark.parametrize("topk_mode", ["hits", "candidates"])
def test_binary_replicas_equal_single_device(ndev, topk_mode):
    xb = _xb()
    x = ck.ref_rademacher(1000, 2000, 3, 4)
    y = np.where(np.random.default_rng(1).random(1000) < 0.5, 1, -1).astype(np.int8)
    cfg = xb.SearchConfig(m=8, l=10, gamma=0.55, seed=7, top_k=50, top_k_mode=topk_mode, threads=1)
    one = xb.Dataset(x).search(y, cfg)
    multi = xb.Dataset(x, devices=[0] * ndev)
    got = multi.search(y, cfg)
    _same(got, one)
    assert got.devices_used == ndev and one.devices_used == 1
    # against the reference as well
    if topk_mode == "hits":
        ok, msg = ck.same_hits(got, ck.ref_search(x, y, cfg))
        assert ok, msg


def test_replicas_stop_after_first_hit_and_explicit_shards():
    """stop_after_first_hit is sequential by definition: the primary runs it
    alone; an explicit rep shard also runs on the primary only."""
    xb = _xb()
    x, y = ck.ref_planted(800, 600, 3, 9, 0.85, 2)
    cfg = xb.SearchConfig(m=8, l=30, gamma=0.8, seed=5, stop_after_first_hit=True, threads=1)
    ds = xb.Dataset(x, devices=[0, 0])
    got = ds.search(y, cfg)
    ok, msg = ck.same_hits(got, ck.ref_search(x, y, cfg))
    assert ok, msg
    assert got.devices_used == 1
    sh = ds.search(y, replace(cfg, stop_after_first_hit=False, rep_begin=3, rep_end=9))
    assert sh.devices_used == 1 and sh.repetitions_run == 2 * 6


@pytest.mark.parametrize("mode,transform", [("continuous_y", "none"), ("continuous_xy", "sign"),
                                            ("continuous_xy", "unbiased")])
def test_continuous_replicas_equal_single_device(mode, transform):
    xb = _xb()
    rng = np.random.default_rng(2)
    n, p = 300, 700
    if mode == "continuous_y":
        x = ck.ref_rademacher(n, p, 9, 9)
    else:
        x = ck.ref_uniform(n, p, 4, 1) if transform == "unbiased" else ck.ref_gaussian(n, p, 4, 1)
    y = rng.standard_normal(n)
    cfg = xb.SearchConfig(m=6, l=9, gamma=0.6, seed=3, mode=mode, transform=transform, top_k=20, threads=1)
    one = xb.Dataset(x).search(y, cfg)
    got = xb.Dataset(x, devices=[0, 0]).search(y, cfg)
    _same(got, one)


def test_real32_dataset_equals_real64_of_the_same_values():
    """x_real32 (half the upload): a float matrix searched as the doubles it
    represents — identical reports to the fp64 dataset of those values, for
    both transforms (the unbiased transform's fp64 rows come from the floats)."""
    xb = _xb()
    rng = np.random.default_rng(8)
    n, p = 257, 900
    v32 = rng.uniform(-1, 1, (p, n)).astype(np.float32)
    v32[rng.random((p, n)) < 0.03] = 0.0
    x32 = xb.RealMatrix(v32, dtype=np.float32)
    x64 = xb.RealMatrix(v32.astype(np.float64))
    y = rng.standard_normal(n)
    for transform in ("sign", "unbiased"):
        cfg = xb.SearchConfig(m=7, l=6, gamma=0.58, seed=9, mode="continuous_xy", transform=transform, top_k=10,
                              threads=1)
        a = xb.Dataset(x32).search(y, cfg)
        b = xb.Dataset(x64).search(y, cfg)
        _same(a, b)
        from tests.test_gpu_parity import compare_continuous
        compare_continuous(ck.hit_tuples(a.hits), ck.hit_tuples(ck.ref_search(x64, y, cfg).hits), cfg.gamma)


def test_bad_device_list_is_a_data_error():
    xb = _xb()
    x = ck.ref_rademacher(64, 10, 1, 1)
    with pytest.raises(xb.DataError):
        xb.Dataset(x, devices=[0, 99])


@pytest.mark.parametrize("topk_mode", ["hits", "candidates"])
def test_binned_replicas_equal_single_device(engine_options, topk_mode):
    """The binned verify on replicas: each shard bins and verifies its own
    runs; binned searches on one device take it in turn (the replicas here
    share device 0), so the shards serialise without deadlock."""
    xb = _xb()
    x = ck.ref_rademacher(5000, 3000, 9, 4)
    y = np.where(np.random.default_rng(2).random(5000) < 0.5, 1, -1).astype(np.int8)
    engine_options(binned=1, binned_wshift=10)
    cfg = xb.SearchConfig(m=10, l=12, gamma=0.52, seed=3, top_k=40, top_k_mode=topk_mode, threads=1,
                          estimate_complexity=False)
    one = xb.Dataset(x).search(y, cfg)
    got = xb.Dataset(x, devices=[0, 0, 0]).search(y, cfg)
    _same(got, one)
    assert got.devices_used == 3
    if topk_mode == "hits":
        ok, msg = ck.same_hits(got, ck.ref_search(x, y, cfg))
        assert ok, msg
