"""GPU exhaustive search (oracle::brute_force_search, oracle.cpp:24-59, 84-91)
against the reference's own brute force: identical pairs, strengths,
histograms and pairs_scanned; the guard; and, at BASELINE config 2 size,
the subset property the reference tests (test_oracle.cpp:28-56): every
positive-pass xyz hit is an oracle hit at the same gamma."""
import numpy as np
import pytest

from tests import checkers as ck

pytestmark = pytest.mark.gpu


def _engine():
    import paper_1610_05108_b200 as xb
    return xb


def _instances():
    rng = np.random.default_rng(5)
    x, y = ck.ref_planted(300, 200, 3, 7, 0.9, 2)
    yield "planted", x, y
    for n in (20, 64, 65, 127):  # few rows: many ties; word boundaries
        xs = rng.choice(np.array([-1, 1], np.int8), size=(n, 90))
        ys = rng.choice(np.array([-1, 1], np.int8), size=n)
        yield f"random_n{n}", _engine().PackedMatrix.from_signs(xs), ys
    xs = rng.choice(np.array([-1, 1], np.int8), size=(130, 150))
    ys = rng.choice(np.array([-1, 0, 1], np.int8), size=130)  # zero responses never agree
    yield "zeros_in_y", _engine().PackedMatrix.from_signs(xs), ys


OPTIONS = [
    dict(gamma=0.6),
    dict(top_k=1),
    dict(top_k=25),
    dict(gamma=0.55, top_k=10),
    dict(histogram_bins=7),
    dict(histogram_bins=100, top_k=3),
    dict(gamma=0.99),
    dict(top_k=0),
]


@pytest.mark.parametrize("kernel", ["tensor", "cuda"])
@pytest.mark.parametrize("opt", OPTIONS, ids=[str(o) for o in OPTIONS])
def test_brute_force_matches_the_reference(opt, kernel, engine_options):
    """Both device kernels: the warp-specialised tcgen05 int8 Gram product
    (default) and the CUDA-core XOR-popcount tiles (the brute_cuda test
    option, an independent cross-check)."""
    if kernel == "cuda":
        engine_options(brute_cuda=1)
    xb = _engine()
    for name, x, y in _instances():
        want_pairs, want_scanned, want_hist = ck.ref_brute_force(x, y, force=True, **opt)
        got = xb.brute_force_search(x, y, force=True, **opt)
        assert got.pairs_scanned == want_scanned, name
        assert [(p.j, p.k, p.strength) for p in got.pairs] == want_pairs, name
        assert got.histogram == want_hist, name


def test_brute_force_guard_like_the_reference():
    xb = _engine()
    rng = np.random.default_rng(1)
    x = xb.PackedMatrix.from_signs(rng.choice(np.array([-1, 1], np.int8), size=(8, 20001)))
    y = np.ones(8, np.int8)
    with pytest.raises(ck.CheckerError) as want:
        ck.ref_brute_force(x, y, top_k=1)
    with pytest.raises(xb.GuardError) as got:
        xb.brute_force_search(x, y, top_k=1)
    assert str(got.value) == str(want.value).split("] ", 1)[1]
    with pytest.raises(xb.DataError, match="response length mismatch"):
        xb.brute_force_search(x, y[:7], top_k=1)
    r = xb.brute_force_search(x, y, top_k=3, force=True)  # 2e8 pairs
    assert r.pairs_scanned == 20001 * 20000 // 2 and len(r.pairs) == 3


def test_xyz_hits_are_oracle_hits_at_config2_size():
    """p = 1e5 (5e9 pairs, far above the reference's guard): the GPU oracle at
    gamma = 0.6 contains every positive-pass hit of the config 2 search, with
    the same strength, and its top pair is at least as strong as any hit."""
    xb = _engine()
    from paper_1610_05108_b200 import synth
    x, y, planted = synth.gwas()
    ds = xb.Dataset(x)
    rep = ds.search(y, xb.SearchConfig(m=16, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False))
    truth = xb.brute_force_search(ds, y, gamma=0.6, force=True)
    assert truth.pairs_scanned == x.n_cols * (x.n_cols - 1) // 2
    oracle = {(p.j, p.k): p.strength for p in truth.pairs}
    pos = [h for h in rep.hits if h.sign > 0]
    assert pos, "config 2 finds its planted pair in the positive pass"
    for h in pos:
        key = (min(h.j, h.k), max(h.j, h.k))
        assert key in oracle and oracle[key] == h.strength
    top = xb.brute_force_search(ds, y, top_k=1, force=True).pairs[0]
    assert top.strength >= max(h.strength for h in pos)


def _weighted_instances():
    rng = np.random.default_rng(9)
    xb = _engine()
    x, _ = ck.ref_planted(300, 200, 3, 7, 0.9, 2)
    yield "planted_gauss", x, rng.standard_normal(300)
    for n in (20, 64, 65, 127):
        xs = rng.choice(np.array([-1, 1], np.int8), size=(n, 90))
        y = rng.standard_normal(n)
        y[::5] = 0.0  # zero responses carry no weight
        yield f"random_n{n}", xb.PackedMatrix.from_signs(xs), y
    xs = rng.choice(np.array([-1, 1], np.int8), size=(100, 120))
    yield "integer_weights_ties", xb.PackedMatrix.from_signs(xs), rng.integers(-3, 4, 100).astype(np.float64)


@pytest.mark.parametrize("opt", OPTIONS, ids=[str(o) for o in OPTIONS])
def test_weighted_brute_force_matches_the_reference(opt):
    """The continuous-response overload (oracle.cpp:93-100): every strength
    bit-identical to scalar_weighted_strength, same selection, ties and
    histogram."""
    xb = _engine()
    for name, x, y in _weighted_instances():
        want_pairs, want_scanned, want_hist = ck.ref_brute_force(x, y, force=True, **opt)
        got = xb.brute_force_search(x, y, force=True, **opt)
        assert got.pairs_scanned == want_scanned, name
        assert [(p.j, p.k, p.strength) for p in got.pairs] == want_pairs, name
        assert got.histogram == want_hist, name


def test_weighted_brute_force_guard_and_zero_response():
    xb = _engine()
    rng = np.random.default_rng(2)
    x = xb.PackedMatrix.from_signs(rng.choice(np.array([-1, 1], np.int8), size=(8, 20001)))
    with pytest.raises(xb.GuardError):
        xb.brute_force_search(x, np.ones(8), top_k=1)
    small = xb.PackedMatrix.from_signs(rng.choice(np.array([-1, 1], np.int8), size=(8, 30)))
    with pytest.raises(ck.CheckerError, match="zero response vector"):
        ck.ref_brute_force(small, np.zeros(8), top_k=1)
    with pytest.raises(xb.DataError, match="zero response vector"):
        xb.brute_force_search(small, np.zeros(8), top_k=1)
