"""The binned verify (csrc/binned_verify.cuh): the search's pairs bucketed by
(z-side column window, x-side column tile) and verified after the last
batch. It is the default for binary X much larger than L2 (config 4, also
covered at full n and p by tests/test_parity_full.py); here it is forced on
small inputs (engine option `binned`) with small windows, so several windows,
tail tiles, several batches and the region regrow path all run, and compared
with the unmodified reference (oracle/_ref) and with the per-batch verify.
"""
from dataclasses import replace

import numpy as np
import pytest

from tests import checkers as ck

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not ck.ref_available(), reason="oracle/_ref not built")]


def _xb():
    import paper_1610_05108_b200 as xb
    return xb


def _data(n, p, seed):
    x = ck.ref_rademacher(n, p, seed, 3)
    y = np.where(np.random.default_rng(seed).random(n) < 0.5, 1, -1).astype(np.int8)
    return x, y


def _counters(r):
    return (r.repetitions_run, r.aborted_repetitions, r.candidates_enumerated)


# n spans every team shape: 100 rows (1 slice per lane), 3000 (2), 5000 (3), 8000 (4), 10240 (5 = the limit)
@pytest.mark.parametrize("n,p,m,l,gamma,wshift", [
    (100, 2000, 10, 5, 0.62, 9), (3000, 2500, 9, 6, 0.53, 10), (5000, 4000, 10, 8, 0.52, 10),
    (8000, 3000, 10, 5, 0.515, 8), (10240, 3333, 10, 4, 0.515, 11)])
def test_binned_hits_equal_reference(engine_options, n, p, m, l, gamma, wshift):
    xb = _xb()
    x, y = _data(n, p, n + p)
    engine_options(binned=1, binned_wshift=wshift)
    cfg = xb.SearchConfig(m=m, l=l, gamma=gamma, seed=5, top_k=20, estimate_complexity=False, threads=1)
    got = xb.Dataset(x).search(y, cfg)
    ref = ck.ref_search(x, y, cfg)
    ok, msg = ck.same_hits(got, ref)
    assert ok, msg
    assert got.top_k == ref.top_k
    assert _counters(got) == _counters(ref)
    assert len(got.hits) > 0


# every grouping path feeds the binned verify: the hashed partition join (sparse 2^24 space), the
# sorted path with 64-bit keys (M = 40: next to no candidates), the split grouping; n = 64 is one word
@pytest.mark.parametrize("n,p,m,l,gamma", [(3000, 4000, 24, 4, 0.5), (3000, 3000, 40, 3, 0.5),
                                            (64, 3000, 12, 6, 0.7), (2000, 5000, 14, 3, 0.53)])
def test_binned_grouping_paths_equal_reference(engine_options, n, p, m, l, gamma):
    xb = _xb()
    x, y = _data(n, p, 3 * n + p + m)
    engine_options(binned=1, binned_wshift=10)
    cfg = xb.SearchConfig(m=m, l=l, gamma=gamma, seed=9, top_k=15, estimate_complexity=False, threads=1)
    got = xb.Dataset(x).search(y, cfg)
    ref = ck.ref_search(x, y, cfg)
    ok, msg = ck.same_hits(got, ref)
    assert ok, msg
    assert got.top_k == ref.top_k
    assert _counters(got) == _counters(ref)


def test_binned_planted_pair_and_stop_after_first_hit(engine_options):
    xb = _xb()
    x, y = ck.ref_planted(6000, 3000, 11, 2900, 0.8, 9)
    engine_options(binned=1, binned_wshift=10)
    for stop in (False, True):
        cfg = xb.SearchConfig(m=10, l=12, gamma=0.56, seed=3, top_k=5, estimate_complexity=False, threads=1,
                              stop_after_first_hit=stop)
        got = xb.Dataset(x).search(y, cfg)
        ref = ck.ref_search(x, y, cfg)
        ok, msg = ck.same_hits(got, ref)
        assert ok, msg
        assert _counters(got) == _counters(ref)
        assert any({h.j, h.k} == {11, 2900} for h in got.hits)


@pytest.mark.parametrize("batch_entries", [0, 9000])
def test_binned_topk_candidates_equals_per_batch_verify(engine_options, batch_entries):
    """Top-K over all candidates: the windows play the per-batch verify's
    batches (ranks in the first, the running threshold afterwards); the
    result equals the per-batch verify's and the reference's A.10 top-K."""
    xb = _xb()
    x, y = _data(5000, 3000, 77)
    cfg = xb.SearchConfig(m=9, l=10, gamma=0.6, seed=11, top_k=300, top_k_mode="candidates",
                          estimate_complexity=False, threads=1)
    engine_options(binned=-1, batch_entries=batch_entries)
    base = xb.Dataset(x).search(y, cfg)
    engine_options(binned=1, binned_wshift=9)
    got = xb.Dataset(x).search(y, cfg)
    assert got.gamma_effective == base.gamma_effective
    ok, msg = ck.same_hits(got, base)
    assert ok, msg
    assert got.top_k == base.top_k
    assert _counters(got) == _counters(base)
    g, rep, want = ck.ref_topk_candidates(x, y, replace(cfg, top_k_mode="hits"), 300, gamma_start=0.56, step=0.002)
    assert ck.hit_tuples(got.top_hits()) == ck.hit_tuples(want), f"gamma grid stopped at {g}"


def test_binned_region_regrow(engine_options):
    """Window regions far too small: the search sizes them from the counts
    it saw and is redone; the result is unchanged."""
    xb = _xb()
    x, y = _data(4000, 3000, 5)
    cfg = xb.SearchConfig(m=9, l=6, gamma=0.53, seed=2, top_k=10, estimate_complexity=False, threads=1)
    engine_options(binned=-1)
    base = xb.Dataset(x).search(y, cfg)
    engine_options(binned=1, binned_wshift=10, binned_cap=100)
    got = xb.Dataset(x).search(y, cfg)
    ok, msg = ck.same_hits(got, base)
    assert ok, msg
    assert got.top_k == base.top_k
    assert _counters(got) == _counters(base)


def test_binned_guard_aborts(engine_options):
    """Runs over the guard emit no pairs into the windows (their counters
    still count), exactly as the reference aborts them."""
    xb = _xb()
    x, y = _data(5000, 2000, 8)
    engine_options(binned=1, binned_wshift=9)
    cfg = xb.SearchConfig(m=5, l=6, gamma=0.52, seed=4, top_k=10, estimate_complexity=False, threads=1,
                          max_candidates_per_rep=10 ** 12)
    ds = xb.Dataset(x)
    free = ds.search(y, cfg)
    cfg = replace(cfg, max_candidates_per_rep=free.candidates_enumerated // free.repetitions_run)  # the mean |E_r|
    got = ds.search(y, cfg)
    ref = ck.ref_search(x, y, cfg)
    ok, msg = ck.same_hits(got, ref)
    assert ok, msg
    assert _counters(got) == _counters(ref)
    assert 0 < got.aborted_repetitions < got.repetitions_run


def test_binned_overflow_list_in_topk_mode(engine_options):
    """Small window / bucket regions: part of every window's pairs go to the
    overflow list (verified by the plain gather, the last top-K phase), the
    rest through the bins; the top-K over all candidates is unchanged."""
    xb = _xb()
    x, y = _data(6000, 2500, 21)
    cfg = xb.SearchConfig(m=9, l=8, gamma=0.6, seed=13, top_k=200, top_k_mode="candidates",
                          estimate_complexity=False, threads=1)
    engine_options(binned=-1)
    base = xb.Dataset(x).search(y, cfg)
    engine_options(binned=1, binned_wshift=9, binned_cap=400)
    ds = xb.Dataset(x)
    for _ in range(2):  # the first search regrows the overflow list; the second runs with it
        got = ds.search(y, cfg)
        assert got.gamma_effective == base.gamma_effective
        ok, msg = ck.same_hits(got, base)
        assert ok, msg
        assert got.top_k == base.top_k
        assert _counters(got) == _counters(base)


@pytest.mark.parametrize("mode", ["hits", "candidates"])
def test_binned_one_pass_join_with_aborted_runs(engine_options, mode):
    """The one-pass partition join (|E_r| counted while the pairs are
    emitted) forced where about half the runs go over the guard: their pairs
    are dropped when binned, counters and hits equal the reference's."""
    xb = _xb()
    x, y = _data(5000, 3000, 31)
    engine_options(binned=1, binned_wshift=10, grouping="part", one_pass_join=1)
    cfg = xb.SearchConfig(m=8, l=8, gamma=0.53, seed=6, top_k=25, top_k_mode=mode, estimate_complexity=False,
                          threads=1, max_candidates_per_rep=10 ** 12)
    ds = xb.Dataset(x)
    free = ds.search(y, cfg)
    cfg = replace(cfg, max_candidates_per_rep=free.candidates_enumerated // free.repetitions_run)
    got = ds.search(y, cfg)
    assert 0 < got.aborted_repetitions < got.repetitions_run
    engine_options(one_pass_join=0, binned=-1)
    base = xb.Dataset(x).search(y, cfg)
    ok, msg = ck.same_hits(got, base)
    assert ok, msg
    assert got.top_k == base.top_k and _counters(got) == _counters(base)
    if mode == "hits":
        ok, msg = ck.same_hits(got, ck.ref_search(x, y, cfg))
        assert ok, msg


@pytest.mark.parametrize("mode", ["hits", "candidates"])
def test_binned_fixed_capacity_partitions(engine_options, mode):
    """The keyless partition pass without its count pass (fixed-capacity
    regions of 4-byte records, config 4's default): equal to the counted pass
    and to the reference; a capacity the partitions overflow is flagged on the
    device and the search redone counted."""
    xb = _xb()
    x, y = _data(5000, 6000, 47)
    cfg = xb.SearchConfig(m=12, l=6, gamma=0.525, seed=8, top_k=25, top_k_mode=mode, estimate_complexity=False,
                          threads=1)
    engine_options(binned=1, binned_wshift=11, grouping="part", part_fixed=-1)
    counted = xb.Dataset(x).search(y, cfg)
    engine_options(part_fixed=0)
    fixed = xb.Dataset(x).search(y, cfg)
    engine_options(part_fixed=8)  # 8 records per partition: every partition overflows
    ds = xb.Dataset(x)
    redone = ds.search(y, cfg)
    engine_options(part_fixed=0)
    again = ds.search(y, cfg)  # one overflow does not switch the dataset to counting
    for got in (fixed, redone, again):
        ok, msg = ck.same_hits(got, counted)
        assert ok, msg
        assert got.top_k == counted.top_k and _counters(got) == _counters(counted)
    assert len(counted.hits) > 0
    assert redone.attempts == fixed.attempts + 1 and again.attempts == fixed.attempts
    if mode == "hits":
        ok, msg = ck.same_hits(fixed, ck.ref_search(x, y, cfg))
        assert ok, msg
