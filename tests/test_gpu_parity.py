"""GPU parity: the CUDA engine (libxyzb.so, through its C ABI) against the
reference's golden fixtures and the CPU restatement (oracle/liboracle.so).

Bars (north_star): bit-exact keys, candidate sets, integer strengths, hit
lists and top-K for +-1 data; strengths within 1e-5 relative for the
continuous modes (X held in fp32 on the device), with pairs inside the
+-1e-5*gamma band of the threshold treated as don't-care.
"""
import os

import numpy as np
import pytest

from tests import checkers as ck
from tests.helpers import GOLDEN, expected_hits, golden_names, load_case, report_hits

pytestmark = pytest.mark.gpu

REL_TOL = 1e-5  # continuous modes (fp32 X on device), north_star tolerance

SEARCH_CASES = [n for n in golden_names() if n.split("_")[0] in ("bin", "cfg1", "cy", "cxy")]


def _engine():
    import paper_1610_05108_b200 as xb
    return xb


def compare_continuous(got, want_hits, gamma, tol=REL_TOL):
    """Hit lists equal up to strength tolerance; pairs within the tolerance
    band around gamma may be present on one side only."""
    band = tol * gamma
    gi = {(h[0], h[1], h[3], h[4]): h[2] for h in got}
    wi = {(h[0], h[1], h[3], h[4]): h[2] for h in want_hits}
    for key, s in wi.items():
        if key in gi:
            assert abs(gi[key] - s) <= tol * abs(s), (key, gi[key], s)
        else:
            assert abs(s - gamma) <= band, f"missing hit {key} s={s}"
    for key, s in gi.items():
        if key not in wi:
            assert abs(s - gamma) <= band, f"extra hit {key} s={s}"
    # order of the common hits is identical
    common_g = [k for k in gi if k in wi]
    common_w = [k for k in wi if k in gi]
    assert common_g == common_w


@pytest.mark.parametrize("grouping", ["auto", "part", "sort", "merge_large"])
@pytest.mark.parametrize("name", SEARCH_CASES)
def test_search_matches_reference_fixture(name, grouping, engine_options):
    """All grouping paths: the engine's choice by M (two CTAs per run
    splitting the 16-bit shared bucket table for 4 <= M <= 16, the partition
    pass + per-(run, partition) tables, ...), the partition path forced, the
    per-run cluster radix sort forced, and the multi-kernel merge."""
    if grouping in ("sort", "part"):
        engine_options(grouping=grouping)
    if grouping == "merge_large":  # the multi-kernel merge instead of the single-CTA one
        engine_options(merge_large=1)
    xb = _engine()
    x, y, cfg, z = load_case(name)
    rep = xb.Dataset(x).search(y, cfg)
    assert rep.repetitions_run == int(z["repetitions_run"])
    assert rep.aborted_repetitions == int(z["aborted_repetitions"])
    assert rep.candidates_enumerated == int(z["candidates_enumerated"])
    assert rep.gamma0 == float(z["gamma0"])
    if cfg.mode == "binary":
        assert report_hits(rep) == expected_hits(z)  # bit-exact
        assert rep.top_k == z["top_k"].tolist()
        assert rep.estimated_c == float(z["estimated_c"])
    else:
        compare_continuous(report_hits(rep), expected_hits(z), cfg.gamma)
        if cfg.estimate_complexity:  # the strength sample is bit-exact in every mode (reference order, no FMA)
            assert rep.estimated_c == float(z["estimated_c"])
    # engine counter = the restatement's canonical count; >= the reference's deduplicated count
    orc = ck.oracle_search(x, y, cfg)
    assert rep.verified_pairs == orc.verified_pairs
    assert rep.verified_pairs >= int(z["candidates_checked"]) or rep.aborted_repetitions > 0
    assert rep.kernel_launches > 0


def test_project_keys_match_reference_fixture():
    xb = _engine()
    z = np.load(os.path.join(GOLDEN, "projection.npz"))
    x = xb.PackedMatrix(int(z["n"]), int(z["p"]), z["x_words"])
    ds = xb.Dataset(x)
    for t in range(int(z["count"])):
        draw = z[f"draw{t}"].astype(np.uint32)
        assert ds.project_keys(draw).tolist()[0] == z[f"keys{t}"].tolist()


def test_project_keys_random_vs_oracle():
    xb = _engine()
    rng = np.random.default_rng(7)
    for n, p in ((1, 5), (63, 70), (64, 33), (65, 129), (1000, 2000)):
        x = ck.ref_rademacher(n, p, n + p, 1)
        ds = xb.Dataset(x)
        for m in (1, 8, 31, 32, 33, 64):
            draws = rng.integers(0, n, (3, m)).astype(np.uint32)
            assert np.array_equal(ds.project_keys(draws), ck.oracle_project_keys(x, draws))


def test_equal_pairs_fig2_and_random():
    xb = _engine()
    z = np.load(os.path.join(GOLDEN, "equal_pairs_fig2.npz"))
    pairs, total = xb.equal_pairs(z["x_keys"], z["z_keys"])
    assert total == 7 and pairs.tolist() == z["pairs"].tolist()
    z = np.load(os.path.join(GOLDEN, "equal_pairs_random.npz"))
    for t in range(int(z["count"])):
        pairs, total = xb.equal_pairs(z[f"x{t}"], z[f"z{t}"])
        assert total == int(z[f"total{t}"]) and pairs.tolist() == z[f"pairs{t}"].tolist()
    # edge cases (test_pair_search.cpp:56-70): disjoint, all identical, wide keys
    pairs, total = xb.equal_pairs(np.array([1, 2, 3], np.uint64), np.array([4, 5, 6], np.uint64))
    assert total == 0 and len(pairs) == 0
    pairs, total = xb.equal_pairs(np.full(17, 9, np.uint64), np.full(17, 9, np.uint64))
    assert total == 17 * 17
    big = np.array([2**64 - 1, 2**63, 5, 2**64 - 1], np.uint64)
    pairs, total = xb.equal_pairs(big, big[::-1].copy())
    want, wt = ck.oracle_equal_pairs(big, big[::-1].copy())
    assert total == wt and pairs.tolist() == want.tolist()


@pytest.mark.parametrize("mode", ["binary", "continuous_y", "continuous_xy_sign", "continuous_xy_unbiased"])
def test_pair_strengths_vs_oracle(mode):
    xb = _engine()
    rng = np.random.default_rng(11)
    n, p = 333, 40
    pairs = rng.integers(0, p, (200, 2)).astype(np.uint32)
    if mode.startswith("continuous_xy"):
        x = ck.ref_uniform(n, p, 5, 5)
        y = rng.normal(size=n)
        tr = mode.split("_")[-1]
        cfg = xb.SearchConfig(mode="continuous_xy", transform=tr)
        want = ck.oracle_pair_strengths(x, y, 2, 1 if tr == "sign" else 2, pairs)
        got = xb.Dataset(x).pair_strengths(y, cfg, pairs)
        np.testing.assert_allclose(got, want, rtol=REL_TOL)
    else:
        x = ck.ref_rademacher(n, p, 5, 5)
        if mode == "binary":
            y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
            cfg = xb.SearchConfig(mode="binary")
            want = ck.oracle_pair_strengths(x, y, 0, 0, pairs)
            got = xb.Dataset(x).pair_strengths(y, cfg, pairs)
            assert np.array_equal(got, want)  # exact integer arithmetic
        else:
            y = rng.normal(size=n)
            y[::7] = 0.0
            cfg = xb.SearchConfig(mode="continuous_y")
            want = ck.oracle_pair_strengths(x, y, 1, 0, pairs)
            got = xb.Dataset(x).pair_strengths(y, cfg, pairs)
            np.testing.assert_allclose(got, want, rtol=1e-12)


@pytest.mark.parametrize("mode", ["binary", "continuous_y", "sign", "unbiased", "sign_f32", "unbiased_f32"])
def test_pair_strengths_bit_exact_vs_reference(mode):
    """xyzb_pair_strengths evaluates each pair in the reference's own order
    with no fused multiply-add: bit-identical to interaction_strength /
    weighted_interaction_strength / the continuous-XY strength on the host
    (fp64 datasets from x_real, and x_real32 datasets, whose values the
    reference gets as doubles)."""
    xb = _engine()
    rng = np.random.default_rng(12)
    n, p = 777, 300
    pairs = rng.integers(0, p, (5000, 2)).astype(np.uint32)
    if mode in ("binary", "continuous_y"):
        x = ck.ref_rademacher(n, p, 7, 7)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8) if mode == "binary" else rng.normal(size=n)
        m, t = (0, 0) if mode == "binary" else (1, 0)
        cfg = xb.SearchConfig(mode="binary" if mode == "binary" else "continuous_y")
        ds = xb.Dataset(x)
    else:
        tr = mode.split("_")[0]
        xv = rng.uniform(-1, 1, (p, n))
        xv[rng.random(xv.shape) < 0.05] = 0.0
        if mode.endswith("f32"):
            x = xb.RealMatrix(xv.astype(np.float32), dtype=np.float32)
        else:
            x = xb.RealMatrix(xv)
        y = rng.normal(size=n)
        m, t = 2, (1 if tr == "sign" else 2)
        cfg = xb.SearchConfig(mode="continuous_xy", transform=tr)
        ds = xb.Dataset(x)
    got = ds.pair_strengths(y, cfg, pairs)
    want = ck.ref_pair_strengths(x, y, m, t, pairs if m else pairs[:, ::-1].copy())
    assert np.array_equal(got, want), np.max(np.abs(got - want))


def test_binary_random_sweep_vs_oracle():
    """Bit-exact hit lists over word-boundary n, M up to 64 (u64 keys), guards."""
    xb = _engine()
    rng = np.random.default_rng(99)
    for t in range(24):
        n = int(rng.choice([1, 2, 63, 64, 65, 127, 300]))
        p = int(rng.integers(2, 160))
        m = int(rng.choice([1, 2, 3, 5, 8, 20, 33, 40, 64]))
        x = ck.ref_rademacher(n, p, 900 + t, 1)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        cfg = xb.SearchConfig(m=m, l=int(rng.integers(1, 6)), gamma=float(rng.choice([0.5, 0.55, 0.6, 0.75, 1.0])),
                              seed=t, search_negatives=bool(rng.random() < 0.8),
                              max_candidates_per_rep=int(rng.choice([0, 0, 50, p])), threads=1,
                              strength_sample_size=int(rng.integers(1, 400)), top_k=int(rng.choice([0, 5, 1000])))
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, (t, msg)
        assert (got.repetitions_run, got.aborted_repetitions, got.candidates_enumerated, got.verified_pairs,
                got.estimated_c, got.top_k) == (want.repetitions_run, want.aborted_repetitions,
                                                want.candidates_enumerated, want.verified_pairs, want.estimated_c,
                                                want.top_k), t


def test_binary_matches_live_reference_cfg1_variants():
    xb = _engine()
    x, y = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    ds = xb.Dataset(x)
    for m, g in ((8, 0.55), (6, 0.6), (12, 0.52)):
        cfg = xb.SearchConfig(m=m, l=10, gamma=g, seed=7, threads=1, top_k=10, estimate_complexity=False)
        got, want = ds.search(y, cfg), ck.ref_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, msg
        assert got.top_k == want.top_k
        assert (got.candidates_enumerated, got.aborted_repetitions) == (want.candidates_enumerated,
                                                                       want.aborted_repetitions)
    # planted pair (5,17) 1-based is recovered
    rep = ds.search(y, xb.SearchConfig(m=8, l=10, gamma=0.6, seed=7, top_k=10))
    assert any((min(h.j, h.k), max(h.j, h.k)) == (4, 16) for h in rep.hits)


@pytest.mark.parametrize("grouping", ["auto", "part", "sort"])
def test_multi_batch_and_hit_regrow_are_invisible(engine_options, grouping):
    """Batching and hit-buffer regrowth must not change anything (the GPU
    analogue of test_search.cpp:275-295, hit lists independent of threads)."""
    xb = _engine()
    x, y = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    cfg = xb.SearchConfig(m=8, l=10, gamma=0.55, seed=7, top_k=10)
    base = xb.Dataset(x).search(y, cfg)
    if grouping in ("sort", "part"):
        engine_options(grouping=grouping)
    # three runs per batch, a shorter last batch; every buffer regrows
    engine_options(batch_entries=6000, hit_cap=7, item_cap=5, pair_cap=100)
    other = xb.Dataset(x).search(y, cfg)
    assert report_hits(other) == report_hits(base)
    assert other.top_k == base.top_k
    assert (other.candidates_enumerated, other.verified_pairs, other.estimated_c) == (
        base.candidates_enumerated, base.verified_pairs, base.estimated_c)


def test_sharded_runs_merge_to_the_full_search():
    """Run sharding (multi-GPU layout) merged through the ABI equals
    the unsharded search, for several shard counts."""
    import ctypes as C
    xb = _engine()
    x, y = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    ds = xb.Dataset(x)
    cfg = xb.SearchConfig(m=8, l=10, gamma=0.55, seed=7, top_k=25, estimate_complexity=False)
    full = ds.search(y, cfg)
    for G in (2, 3, 4, 10):
        parts = []
        bounds = [1 + (cfg.l * g) // G for g in range(G + 1)]
        for g in range(G):
            sub = xb.SearchConfig(**{**cfg.__dict__, "rep_begin": bounds[g], "rep_end": bounds[g + 1]})
            parts.append(ds.search_raw(y, sub))
        try:
            merged = ds.merge(parts, cfg)
        finally:
            for r in parts:
                ds.free_result(r)
        assert report_hits(merged) == report_hits(full), G
        assert merged.top_k == full.top_k
        assert merged.candidates_enumerated == full.candidates_enumerated
        assert merged.repetitions_run == full.repetitions_run


def test_data_errors_like_the_reference():
    xb = _engine()
    x, y = ck.ref_planted(64, 12, 0, 1, 1.0, 7)
    ds = xb.Dataset(x)
    with pytest.raises(xb.DataError):
        ds.search(y, xb.SearchConfig(m=0))
    with pytest.raises(xb.DataError):
        ds.search(y, xb.SearchConfig(m=65))
    with pytest.raises(xb.DataError):
        ds.search(y, xb.SearchConfig(gamma=0.0))
    with pytest.raises(xb.DataError):
        ds.search(y, xb.SearchConfig(l=0))
    bad = y.copy()
    bad[3] = 0
    with pytest.raises(xb.DataError):
        ds.search(bad, xb.SearchConfig())
    with pytest.raises(xb.DataError):
        ds.search(y, xb.SearchConfig(transform="sign"))
    with pytest.raises(xb.DataError):
        ds.search(np.zeros(64), xb.SearchConfig(mode="continuous_y"))
    with pytest.raises(xb.DataError):
        xb.xyz_search(x, y[:10], xb.SearchConfig())
    big = xb.RealMatrix(np.full((2, 4), 2.0))
    with pytest.raises(xb.DataError):
        xb.Dataset(big).search(np.ones(4), xb.SearchConfig(mode="continuous_xy", transform="unbiased"))


def test_continuous_modes_random_vs_oracle():
    xb = _engine()
    rng = np.random.default_rng(5)
    for t in range(6):
        n, p = int(rng.integers(30, 400)), int(rng.integers(5, 120))
        if t % 2 == 0:
            x = ck.ref_rademacher(n, p, t, 8)
            y = rng.normal(size=n)
            y[rng.random(n) < 0.1] = 0.0
            cfg = xb.SearchConfig(m=int(rng.integers(2, 7)), l=4, gamma=0.56, seed=t, mode="continuous_y",
                                  threads=1, strength_sample_size=200, top_k=9)
        else:
            xr = ck.ref_uniform(n, p, t, 8)
            v = xr.values.copy()
            v[rng.random(v.shape) < 0.05] = 0.0
            x = xb.RealMatrix(v)
            y = rng.normal(size=n)
            cfg = xb.SearchConfig(m=int(rng.integers(2, 6)), l=4, gamma=0.55, seed=t, mode="continuous_xy",
                                  transform="unbiased" if t % 4 == 1 else "sign", threads=1,
                                  strength_sample_size=200, top_k=9)
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        assert got.candidates_enumerated == want.candidates_enumerated, t  # keys bit-exact
        assert got.aborted_repetitions == want.aborted_repetitions
        compare_continuous(report_hits(got), report_hits(want), cfg.gamma)


def test_gwas_full_size_properties():
    """BASELINE config 2 at full size (n=4000, p=1e5, M=16, L=100): the oracle
    cannot finish here, so check size-independent properties: every hit's
    strength recomputed exactly on the host, the A.8 order and dedup rules,
    top-K consistency, and shard-merge equality."""
    from paper_1610_05108_b200 import synth
    xb = _engine()
    x, y, planted = synth.gwas()
    ds = xb.Dataset(x)
    cfg = xb.SearchConfig(m=16, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False)
    rep = ds.search(y, cfg)
    assert rep.repetitions_run == 200 and rep.runs_executed == 200
    assert rep.verified_pairs > 0
    # exact strengths
    pairs = np.array([[h.j, h.k] for h in rep.hits], np.uint32).reshape(-1, 2)
    if len(pairs):
        xw = x.words
        from paper_1610_05108_b200.matrix import pack_signs
        yw = pack_signs(y)
        agree = np.array([int(np.unpackbits((xw[j] ^ xw[k] ^ yw).view(np.uint8)).sum()) for j, k in pairs])
        n = x.n_rows
        for h, a in zip(rep.hits, agree):
            s = a / n if h.sign > 0 else (n - a) / n
            assert h.strength == s and s >= cfg.gamma
    # dedup: one hit per (min, max, sign); order by (sign pass, rep)
    keys = [(min(h.j, h.k), max(h.j, h.k), h.sign) for h in rep.hits]
    assert len(keys) == len(set(keys))
    ordr = [(0 if h.sign > 0 else 1, h.found_at_repetition) for h in rep.hits]
    assert ordr == sorted(ordr)
    # a planted interaction is found (the others are weaker than gamma=0.6 marginally)
    found = {(min(h.j, h.k), max(h.j, h.k)) for h in rep.hits}
    assert len(found & {tuple(p) for p in planted.tolist()}) >= 1
    # top-K: strength-descending with the A.10 tie-break
    top = rep.top_hits()
    ts = [(-h.strength, min(h.j, h.k), max(h.j, h.k), -h.sign) for h in top]
    assert ts == sorted(ts)


def test_xyz1_file_ingest_matches_in_memory_and_reference_errors(tmp_path):
    """xyzb_dataset_open streams the reference's on-disk format (written by the
    reference's own write_dataset) straight to HBM; searches are identical to
    the in-memory dataset; malformed files fail with read_dataset's messages."""
    xb = _engine()
    x, y = ck.ref_planted(300, 120, 3, 7, 0.95, 2)
    f = tmp_path / "x.xyz"
    ck.ref_write_dataset(f, x)
    cfg = xb.SearchConfig(m=6, l=8, gamma=0.6, seed=3, top_k=10)
    a = xb.Dataset.open(f).search(y, cfg)
    b = xb.Dataset(x).search(y, cfg)
    assert report_hits(a) == report_hits(b) and a.top_k == b.top_k
    xr = ck.ref_uniform(50, 9, 4, 4)
    fr = tmp_path / "r.xyz"
    ck.ref_write_dataset(fr, xr)
    yr = np.random.default_rng(3).normal(size=50)
    cr = xb.SearchConfig(m=3, l=4, gamma=0.55, seed=1, mode="continuous_xy", transform="sign")
    assert report_hits(xb.Dataset.open(fr).search(yr, cr)) == report_hits(xb.Dataset(xr).search(yr, cr))
    raw = f.read_bytes()
    bad = {
        "magic": b"XYZ2" + raw[4:],
        "kind": raw[:4] + b"\x07" + raw[5:],
        "dims": raw[:8] + (0).to_bytes(8, "little") + raw[16:],
        "truncated": raw[:-5],
        "trailing": raw + b"\x00",
        "padding": raw[:24 + 8 * 4] + (1 << 63).to_bytes(8, "little") + raw[24 + 8 * 5:],  # last word of column 0
    }
    for name, blob in bad.items():
        g = tmp_path / f"bad_{name}.xyz"
        g.write_bytes(blob)
        with pytest.raises(ck.CheckerError) as want:
            ck.ref_read_dataset(g)
        with pytest.raises(xb.DataError) as got:
            xb.Dataset.open(g)
        assert str(got.value) == str(want.value).split("] ", 1)[1], name
    with pytest.raises(xb.DataError):
        xb.Dataset.open(tmp_path / "missing.xyz")


@pytest.mark.parametrize("grouping", ["auto", "part"])
def test_bucket_above_16_bits_falls_back_exactly(grouping, engine_options):
    """p > 65535 with 70000 identical (monomorphic) columns: one bucket holds
    more columns than a 16-bit shared counter can; the CTA grouping redoes
    such a run with 32-bit counters. Hits and counters equal the reference."""
    if grouping == "part":
        engine_options(grouping=grouping)
    xb = _engine()
    rng = np.random.default_rng(11)
    n, p_const, p_rand = 128, 70000, 300
    signs = np.ones((n, p_const + p_rand), np.int8)
    signs[:, p_const:] = rng.choice(np.array([-1, 1], np.int8), size=(n, p_rand))
    x = xb.PackedMatrix.from_signs(signs)
    y = rng.choice(np.array([-1, 1], np.int8), size=n)
    for m, l, g in ((16, 3, 0.6), (14, 2, 0.62)):
        cfg = xb.SearchConfig(m=m, l=l, gamma=g, seed=5, threads=1, top_k=20, estimate_complexity=False)
        got, want = xb.Dataset(x).search(y, cfg), ck.ref_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, msg
        assert got.top_k == want.top_k
        assert (got.candidates_enumerated, got.aborted_repetitions) == (want.candidates_enumerated,
                                                                       want.aborted_repetitions)


def test_dirty_padding_bits_are_rejected_on_upload():
    """The PackedMatrix invariant (packed_matrix.hpp:10-14): bits above row
    n-1 of a column's last word must be zero; checked on the device after the
    upload, naming the first offending column."""
    xb = _engine()
    x, _ = ck.ref_planted(100, 40, 3, 7, 0.9, 1)
    words = x.words.copy()
    words[3, -1] |= np.uint64(1) << np.uint64(63)
    words[17, -1] |= np.uint64(1) << np.uint64(40)
    with pytest.raises(xb.DataError, match="padding bits of column 3 are not zero"):
        xb.Dataset(xb.PackedMatrix(100, 40, words))  # pageable: checked on the host
    import torch
    pin = torch.empty(words.nbytes, dtype=torch.uint8, pin_memory=True)
    pinned = pin.numpy().view(np.uint64).reshape(words.shape)
    pinned[...] = words
    with pytest.raises(xb.DataError, match="padding bits of column 3 are not zero"):
        xb.Dataset(xb.PackedMatrix(100, 40, pinned))  # page-locked: DMA'd, checked on the device
    pinned[...] = x.words
    y = ck.ref_planted(100, 40, 3, 7, 0.9, 1)[1]
    cfg = xb.SearchConfig(m=4, l=6, gamma=0.6, seed=2)
    assert report_hits(xb.Dataset(xb.PackedMatrix(100, 40, pinned)).search(y, cfg)) == report_hits(
        xb.Dataset(x).search(y, cfg))


@pytest.mark.parametrize("grouping", ["auto", "part"])
def test_constant_response_partner_is_the_complement(grouping, engine_options):
    """y constant: in the negative pass c = x-key ^ z-key has every bit set, so
    each key's partner is its complement (no key bit is shared by a key and
    its partner: the two-CTA split reads the partner half through DSMEM)."""
    if grouping == "part":
        engine_options(grouping=grouping)
    xb = _engine()
    x, _ = ck.ref_planted(300, 400, 3, 7, 0.9, 3)
    y = np.ones(300, np.int8)
    for m, g in ((6, 0.6), (10, 0.56)):
        cfg = xb.SearchConfig(m=m, l=5, gamma=g, seed=9, threads=1, top_k=30, estimate_complexity=False)
        got, want = xb.Dataset(x).search(y, cfg), ck.ref_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, msg
        assert got.top_k == want.top_k
        assert (got.candidates_enumerated, got.aborted_repetitions) == (want.candidates_enumerated,
                                                                       want.aborted_repetitions)
        assert len(want.hits) > 0


@pytest.mark.parametrize("grouping", ["auto", "part"])
def test_grouping_kernels_sweep_vs_oracle(grouping, engine_options):
    """The fused group + join kernels (two-CTA split, one CTA, DSMEM cluster)
    over the M range they serve (4..17) and p from a handful of columns to
    2^M-sized tables: bit-exact against the restatement."""
    if grouping == "part":
        engine_options(grouping=grouping)
    xb = _engine()
    rng = np.random.default_rng(7)
    cases = [(4, 3), (5, 40), (6, 700), (8, 2000), (11, 600), (12, 5000), (13, 3000), (14, 9000), (15, 12000),
             (16, 20000), (17, 33000)]
    for t, (m, p) in enumerate(cases):
        n = int(rng.choice([63, 64, 65, 130]))
        x = ck.ref_rademacher(n, p, 300 + t, 2)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        cfg = xb.SearchConfig(m=m, l=2, gamma=0.7, seed=t, threads=1, top_k=20,
                              max_candidates_per_rep=int(rng.choice([0, p])), estimate_complexity=False)
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, (m, p, msg)
        assert (got.aborted_repetitions, got.candidates_enumerated, got.verified_pairs, got.top_k) == (
            want.aborted_repetitions, want.candidates_enumerated, want.verified_pairs, want.top_k), (m, p)


def test_concurrent_searches_on_different_datasets():
    """Host threads driving different datasets (one stream each) concurrently
    get exactly the serial results (the engine's buffers wait on their own
    stream when they return to the shared pool)."""
    from concurrent.futures import ThreadPoolExecutor
    xb = _engine()
    jobs = []
    for t in range(6):
        x, y = ck.ref_planted(400, 1500 + 100 * t, 2, 9, 0.9, 10 + t)
        cfg = xb.SearchConfig(m=8 + t % 3, l=6, gamma=0.56, seed=t, top_k=10)
        jobs.append((x, y, cfg))
    serial = [report_hits(xb.Dataset(x).search(y, cfg)) for x, y, cfg in jobs]

    def run(job):
        x, y, cfg = job
        d = xb.Dataset(x)
        try:
            return report_hits(d.search(y, cfg))
        finally:
            d.close()

    for _ in range(3):
        with ThreadPoolExecutor(3) as ex:
            assert list(ex.map(run, jobs)) == serial


@pytest.mark.parametrize("case", ["dense", "sparse_forced", "constant_y"])
def test_msplit_grouping_vs_oracle(case, engine_options):
    """17 <= M <= 20: one 2^(M-16)-CTA cluster per run (16 CTAs at M = 20).
    Dense tables by default, a sparse run forced onto it, and a constant
    response (c = all ones in the negative pass: partners in other CTAs,
    read through DSMEM). Bit-exact against the restatement."""
    xb = _engine()
    rng = np.random.default_rng(17)
    if case == "dense":  # M = 19, 20 only when forced (the counting sort is faster there)
        engine_options(grouping="msplit")
        cases = [(17, 40000), (18, 70000), (19, 140000), (20, 270000)]
    elif case == "sparse_forced":
        engine_options(grouping="msplit")
        cases = [(18, 3000), (20, 9000)]
    else:
        cases = [(18, 70000), (17, 40000)]
    for t, (m, p) in enumerate(cases):
        n = 64
        x = ck.ref_rademacher(n, p, 500 + t, 3)
        y = np.ones(n, np.int8) if case == "constant_y" else np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        cfg = xb.SearchConfig(m=m, l=2, gamma=0.72, seed=t, threads=1, top_k=20, estimate_complexity=False)
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, (m, p, msg)
        assert (got.aborted_repetitions, got.candidates_enumerated, got.verified_pairs, got.top_k) == (
            want.aborted_repetitions, want.candidates_enumerated, want.verified_pairs, want.top_k), (m, p)


@pytest.mark.parametrize("case", ["dense", "forced_low_m", "constant_y", "guard", "biased"])
def test_partition_grouping_vs_oracle(case, engine_options):
    """The partitioned path (default for M >= 19 with a dense bucket space):
    a partition pass on the top bits of T(v) (T linear, T(c) = e_0, so a key
    and its partner share a partition and are neighbouring local buckets),
    then one CTA per (run, partition). M = 19..22 by default, M = 4..18
    forced, a constant response (c = all ones), runs the guard aborts, and
    heavily biased columns (skewed partitions). Bit-exact against the
    restatement."""
    xb = _engine()
    rng = np.random.default_rng(23)
    guard = None
    if case == "dense":
        cases = [(19, 140000), (20, 270000), (21, 600000), (22, 1100000)]
    elif case == "forced_low_m":
        engine_options(grouping="part")
        cases = [(4, 20), (7, 300), (12, 2000), (13, 5000), (14, 9000), (16, 20000), (18, 70000)]
    elif case == "constant_y":
        cases = [(19, 140000), (20, 270000)]
    elif case == "guard":
        engine_options(grouping="part")
        cases = [(14, 6000), (19, 140000)]
        guard = 1
    else:
        cases = [(20, 270000)]
    for t, (m, p) in enumerate(cases):
        n = 64
        if case == "biased":  # columns with few +1 rows: keys crowd the low buckets
            signs = np.where(rng.random((n, p)) < rng.uniform(0.02, 0.5, p), 1, -1).astype(np.int8)
            x = xb.PackedMatrix.from_signs(signs)
        else:
            x = ck.ref_rademacher(n, p, 900 + t, 3)
        y = np.ones(n, np.int8) if case == "constant_y" else np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        cfg = xb.SearchConfig(m=m, l=2, gamma=0.72, seed=t, threads=1, top_k=20, estimate_complexity=False,
                              max_candidates_per_rep=(p // 8 if guard else 0))
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, (m, p, msg)
        assert (got.aborted_repetitions, got.candidates_enumerated, got.verified_pairs, got.top_k) == (
            want.aborted_repetitions, want.candidates_enumerated, want.verified_pairs, want.top_k), (m, p)


@pytest.mark.parametrize("case", ["sparse", "wide_keys", "constant_y", "guard", "skewed_overflow", "forced_sort"])
def test_hashed_partition_grouping_vs_oracle(case, engine_options):
    """Sparse bucket spaces (2^M > 4p + 1024, M <= 31): the partition pass
    plus one CTA per (run, partition) with an open-addressing hash table in
    shared memory. Covers M up to 31, c = all ones, guard aborts, a skewed
    key distribution whose partitions overflow the table (the search is then
    redone on the sorted path), and the sorted path forced. Bit-exact
    against the restatement."""
    xb = _engine()
    rng = np.random.default_rng(29)
    guard = None
    if case == "sparse":
        cases = [(12, 300), (16, 2000), (20, 50000), (22, 30000)]
    elif case == "wide_keys":
        cases = [(26, 40000), (31, 20000)]
    elif case == "constant_y":
        cases = [(20, 50000), (14, 900)]
    elif case == "guard":
        cases = [(18, 20000)]
        guard = 1
    elif case == "forced_sort":
        engine_options(grouping="sort")
        cases = [(20, 50000)]
    else:
        cases = [(21, 100000)]
    for t, (m, p) in enumerate(cases):
        n = 64
        if case == "skewed_overflow":  # columns with few +1 rows: most keys share their top bits
            signs = np.where(rng.random((n, p)) < rng.uniform(0.01, 0.2, p), 1, -1).astype(np.int8)
            x = xb.PackedMatrix.from_signs(signs)
        else:
            x = ck.ref_rademacher(n, p, 1300 + t, 3)
        y = np.ones(n, np.int8) if case == "constant_y" else np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        cfg = xb.SearchConfig(m=m, l=2, gamma=0.7, seed=t, threads=1, top_k=20, estimate_complexity=False,
                              max_candidates_per_rep=(p // 20 if guard else 0))
        got = xb.Dataset(x).search(y, cfg)
        want = ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(got, want)
        assert ok, (m, p, msg)
        assert (got.aborted_repetitions, got.candidates_enumerated, got.verified_pairs, got.top_k) == (
            want.aborted_repetitions, want.candidates_enumerated, want.verified_pairs, want.top_k), (m, p)


@pytest.mark.parametrize("n", [100, 2000, 3000])
def test_sign_bit_verify_equals_fp32_verify(n, engine_options):
    """The sign transform's bit-plane verify (column sign bits x quantised
    response planes, re-verification within the quantisation bound) reports
    exactly the hits and strengths of the fp32-column verify, with exact
    zeros in X (nonzero masks) and without, for row counts on both sides of
    the register-resident plane path (<= 2048 rows); and matches the
    restatement within the continuous tolerance."""
    xb = _engine()
    rng = np.random.default_rng(n)
    p = 3000
    xv = rng.normal(size=(p, n))
    if n != 2000:
        xv[rng.random((p, n)) < 0.05] = 0.0  # exact zeros: the coin path for keys, nonzero masks here
    y = xv[3] * xv[11] * 0.8 + rng.normal(size=n)
    x = xb.RealMatrix(xv)
    total = 0
    for gamma in (0.52, 0.55):
        cfg = xb.SearchConfig(m=9, l=6, gamma=gamma, seed=4, threads=1, top_k=30, mode="continuous_xy",
                              transform="sign", estimate_complexity=False)
        got = xb.Dataset(x).search(y, cfg)
        engine_options(sign_verify_off=1)
        ref = xb.Dataset(x).search(y, cfg)
        engine_options(sign_verify_off=0)
        assert report_hits(got) == report_hits(ref), (n, gamma)
        assert got.top_k == ref.top_k and got.verified_pairs == ref.verified_pairs
        want = ck.oracle_search(x, y, cfg)
        compare_continuous(report_hits(got), [(h.j, h.k, h.strength, h.found_at_repetition, h.sign)
                                              for h in want.hits], gamma)
        total += len(got.hits)
    assert total > 0


def test_hashed_grouping_batches_and_regrow_are_invisible(engine_options):
    """The hashed partition join under multi-batch runs and forced item /
    pair / hit buffer regrowth gives the unbatched, unregrown result."""
    xb = _engine()
    x, y = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    cfg = xb.SearchConfig(m=14, l=10, gamma=0.55, seed=7, top_k=10)  # 2^14 > 4p + 1024: sparse
    base = xb.Dataset(x).search(y, cfg)
    engine_options(batch_entries=6000, hit_cap=7, item_cap=5, pair_cap=100)
    other = xb.Dataset(x).search(y, cfg)
    assert report_hits(other) == report_hits(base) and other.top_k == base.top_k
    assert (other.candidates_enumerated, other.verified_pairs) == (base.candidates_enumerated, base.verified_pairs)
    want = ck.oracle_search(x, y, cfg)
    ok, msg = ck.same_hits(base, want)
    assert ok, msg


@pytest.mark.parametrize("n", [200, 2000, 2100])
def test_weighted_bit_plane_verify_equals_exact_verify(n, engine_options):
    """Continuous-Y (A9): the bit-plane verify over the pair list (|y|
    quantised to 12-bit planes, exact re-verification within the
    quantisation bound; rows <= 2048) reports exactly the hits and strengths
    of the exact fp64 verify, and matches the reference within 1e-5; above
    2048 rows the item walk runs."""
    xb = _engine()
    rng = np.random.default_rng(n)
    x = ck.ref_rademacher(n, 1500, n, 2)
    y = rng.standard_normal(n)
    y[::9] = 0.0
    total = 0
    for gamma in (0.53, 0.56):
        cfg = xb.SearchConfig(m=8, l=6, gamma=gamma, seed=4, threads=1, top_k=30, mode="continuous_y",
                              estimate_complexity=False)
        got = xb.Dataset(x).search(y, cfg)
        engine_options(sign_verify_off=1)
        ref = xb.Dataset(x).search(y, cfg)
        engine_options(sign_verify_off=0)
        assert report_hits(got) == report_hits(ref), (n, gamma)
        assert got.top_k == ref.top_k and got.verified_pairs == ref.verified_pairs
        compare_continuous(report_hits(got), ck.hit_tuples(ck.ref_search(x, y, cfg).hits), gamma)
        total += len(got.hits)
    assert total > 0
