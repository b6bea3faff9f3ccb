"""Top-K over ALL verified candidates (BASELINE north_star; SURVEY A.10,
§8a A12): the engine's XYZB_TOPK_CANDIDATES mode against the unmodified
reference (oracle/_ref).

Two independent checks per case:
  1. the engine's hit list equals the reference's A.8 hit list at
     gamma = the engine's gamma_effective (the K-th ranked strength), bit for
     bit for +-1 data (order, orientation, strength, repetition, sign);
  2. the engine's top-K equals A.10's gamma-lowering procedure run on the
     reference: lower gamma on a grid until the hit list holds >= K entries,
     then rank by (strength desc, min, max, sign desc).
Continuous modes: strengths within 1e-5 relative, ties inside that band
don't-care (X is fp32 on the device).
"""
from dataclasses import replace

import numpy as np
import pytest

from tests import checkers as ck

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5


def _xb():
    import paper_1610_05108_b200 as xb
    return xb


def _topk_cfg(cfg, k):
    return replace(cfg, top_k=k, top_k_mode="candidates", estimate_complexity=False)


def check_binary(x, y, cfg, k, ds=None, gamma_start=0.6):
    xb = _xb()
    ds = ds or xb.Dataset(x)
    got = ds.search(y, _topk_cfg(cfg, k))
    # 1: the hit list is the reference's A.8 list at gamma_effective
    assert got.gamma_effective > 0
    ref = ck.ref_search(x, y, replace(cfg, gamma=got.gamma_effective, top_k=k, estimate_complexity=False))
    ok, msg = ck.same_hits(got, ref)
    assert ok, msg
    assert got.top_k == ref.top_k
    assert (got.repetitions_run, got.aborted_repetitions, got.candidates_enumerated) == \
        (ref.repetitions_run, ref.aborted_repetitions, ref.candidates_enumerated)
    # 2: A.10 gamma-lowering on the reference
    g, rep, want = ck.ref_topk_candidates(x, y, cfg, k, gamma_start=gamma_start)
    assert ck.hit_tuples(got.top_hits()) == ck.hit_tuples(want), f"gamma grid stopped at {g}"
    assert len(got.top_k) == min(k, len(rep.hits))
    return got


@pytest.mark.parametrize("n,p,m,l,k,neg", [
    (100, 300, 6, 6, 1, True), (257, 400, 8, 5, 7, True), (1000, 2000, 8, 10, 50, True),
    (64, 500, 5, 4, 300, False), (999, 1500, 10, 20, 400, True), (200, 3000, 12, 3, 1000, True)])
def test_topk_candidates_binary_vs_reference(n, p, m, l, k, neg):
    x = ck.ref_rademacher(n, p, n + p + m, 3)
    y = np.where(np.random.default_rng(n).random(n) < 0.5, 1, -1).astype(np.int8)
    cfg = _xb().SearchConfig(m=m, l=l, gamma=0.9, seed=11, search_negatives=neg, threads=1)
    got = check_binary(x, y, cfg, k)
    assert got.verified_pairs > 0


def test_topk_candidates_toy_cfg1():
    """BASELINE config 1 (n=1000, p=2000, M=8, L=10) with K=10: the planted
    pair (5,17) is the top entry."""
    from paper_1610_05108_b200 import synth
    x, y = synth.toy(1000, 2000, 4, 16, 0.9, 1)
    cfg = _xb().SearchConfig(m=8, l=10, gamma=0.55, seed=7, threads=1)
    got = check_binary(x, y, cfg, 10, gamma_start=0.95)
    top = got.top_hits()[0]
    assert (min(top.j, top.k), max(top.j, top.k)) == (4, 16)


def test_topk_candidates_guard_aborts_and_batches(engine_options):
    """Aborted runs contribute nothing; many small batches exercise the
    running threshold and the prune between batches."""
    engine_options(batch_entries=900)
    x = ck.ref_rademacher(300, 450, 5, 9)
    y = np.where(np.arange(300) % 3 == 0, 1, -1).astype(np.int8)
    cfg = _xb().SearchConfig(m=5, l=30, gamma=0.9, seed=3, max_candidates_per_rep=6300, threads=1)
    got = check_binary(x, y, cfg, 120)
    assert 0 < got.aborted_repetitions < got.repetitions_run


def test_topk_candidates_duplicates_dominate():
    """A strong planted pair is a candidate in most runs: the raw top of every
    batch is dominated by its duplicates (the distinct count decides)."""
    x, y = ck.ref_planted(500, 800, 10, 20, 0.97, 4)
    cfg = _xb().SearchConfig(m=10, l=60, gamma=0.9, seed=5, threads=1)
    got = check_binary(x, y, cfg, 40, gamma_start=0.99)
    assert (min(got.top_hits()[0].j, got.top_hits()[0].k), max(got.top_hits()[0].j, got.top_hits()[0].k)) == (10, 20)


def test_topk_candidates_shards_merge_equal_unsharded():
    xb = _xb()
    x = ck.ref_rademacher(640, 1200, 17, 2)
    y = np.where(np.random.default_rng(3).random(640) < 0.4, 1, -1).astype(np.int8)
    cfg = _topk_cfg(xb.SearchConfig(m=7, l=12, gamma=0.9, seed=21, threads=1), 200)
    ds = xb.Dataset(x)
    whole = ds.search(y, cfg)
    from paper_1610_05108_b200 import parallel
    for world in (2, 3, 5):
        parts = [ds.search_raw(y, parallel.shard_config(cfg, r, world)) for r in range(world)]
        try:
            merged = ds.merge(parts, cfg)
        finally:
            for r in parts:
                ds.free_result(r)
        assert ck.hit_tuples(merged.hits) == ck.hit_tuples(whole.hits)
        assert merged.top_k == whole.top_k and merged.gamma_effective == whole.gamma_effective


def _compare_continuous_topk(got, ref_hits, k):
    """Top-K lists equal up to 1e-5 relative strengths; entries whose strength
    lies within the tolerance of the K-th strength may differ (near-ties)."""
    sk = got.top_hits()[-1].strength
    band = REL_TOL * sk
    g = {(h.j, h.k, h.found_at_repetition, h.sign): h.strength for h in got.top_hits()}
    w = {(h.j, h.k, h.found_at_repetition, h.sign): h.strength for h in ck.topk_a10(ref_hits, k)}
    for key, s in w.items():
        if key in g:
            assert abs(g[key] - s) <= REL_TOL * abs(s), (key, g[key], s)
        else:
            assert abs(s - sk) <= band, f"missing top-K entry {key} s={s} (K-th {sk})"
    for key, s in g.items():
        if key not in w:
            assert abs(s - sk) <= band, f"extra top-K entry {key} s={s} (K-th {sk})"


@pytest.mark.parametrize("mode,transform", [("continuous_y", "none"), ("continuous_xy", "sign"),
                                            ("continuous_xy", "unbiased")])
def test_topk_candidates_continuous_vs_reference(mode, transform):
    xb = _xb()
    rng = np.random.default_rng(5)
    n, p, k = 400, 900, 150
    if mode == "continuous_y":
        x = ck.ref_rademacher(n, p, 8, 8)
        y = rng.standard_normal(n)
        y[::37] = 0.0
    else:
        x = ck.ref_uniform(n, p, 6, 2) if transform == "unbiased" else ck.ref_gaussian(n, p, 6, 2)
        y = rng.standard_normal(n)
    if transform == "sign":
        xv = x.values.copy()
        xv[rng.random(xv.shape) < 0.05] = 0.0
        x = xb.RealMatrix(xv)
    cfg = xb.SearchConfig(m=6, l=8, gamma=0.9, seed=13, mode=mode, transform=transform, threads=1)
    got = xb.Dataset(x).search(y, _topk_cfg(cfg, k))
    assert len(got.top_k) == k
    g, rep, _ = ck.ref_topk_candidates(x, y, cfg, k, gamma_start=0.7)
    _compare_continuous_topk(got, rep.hits, k)
    # the hit list: every reference hit at gamma_effective (outside the band) is an engine hit
    ref = ck.ref_search(x, y, replace(cfg, gamma=got.gamma_effective, estimate_complexity=False))
    from tests.test_gpu_parity import compare_continuous
    compare_continuous(ck.hit_tuples(got.hits), ck.hit_tuples(ref.hits), got.gamma_effective)


def test_topk_candidates_rejects_bad_config():
    xb = _xb()
    x = ck.ref_rademacher(64, 50, 1, 1)
    y = np.ones(64, np.int8)
    ds = xb.Dataset(x)
    with pytest.raises(xb.DataError):
        ds.search(y, replace(xb.SearchConfig(m=4, l=2), top_k=0, top_k_mode="candidates"))
    with pytest.raises(xb.DataError):
        ds.search(y, replace(xb.SearchConfig(m=4, l=2), top_k=5, top_k_mode="candidates", stop_after_first_hit=True))
