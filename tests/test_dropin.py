"""The drop-in: the reference's own C++ core with search.cpp replaced by the
GPU shim (build/dropin/libxyz_core_gpu.so). The reference's unchanged callers
— here lasso_path (lasso.cpp:447-597), whose KKT screen calls xyz_search —
run on the B200 engine, and must agree with the all-CPU reference build
(oracle/_ref/libxyzref.so) driven through the same harness."""
import numpy as np
import pytest

from tests import checkers as ck
from tests.helpers import expected_hits, golden_names, load_case, report_hits

pytestmark = pytest.mark.gpu

BINARY_CASES = [n for n in golden_names() if n.split("_")[0] in ("bin", "cfg1")]


@pytest.mark.parametrize("name", BINARY_CASES)
def test_dropin_xyz_search_is_the_reference(name):
    """xyz::xyz_search through the shim reproduces the reference fixtures."""
    x, y, cfg, z = load_case(name)
    rep = ck.dropin_search(x, y, cfg)
    assert report_hits(rep) == expected_hits(z)
    assert (rep.repetitions_run, rep.aborted_repetitions, rep.candidates_enumerated, rep.estimated_c) == (
        int(z["repetitions_run"]), int(z["aborted_repetitions"]), int(z["candidates_enumerated"]),
        float(z["estimated_c"]))


def test_dropin_validation_messages_match():
    from paper_1610_05108_b200.report import SearchConfig
    x, y = ck.ref_planted(64, 12, 0, 1, 1.0, 7)
    for cfg in (SearchConfig(m=0), SearchConfig(gamma=0.0), SearchConfig(transform="sign")):
        with pytest.raises(ck.CheckerError) as a:
            ck.ref_search(x, y, cfg)
        with pytest.raises(ck.CheckerError) as b:
            ck.dropin_search(x, y, cfg)
        assert a.value.code == b.value.code == 3
        assert str(a.value) == str(b.value)


def _compare_fits(gpu, cpu, tol=1e-4):
    assert len(gpu) == len(cpu)
    for g, c in zip(gpu, cpu):
        assert abs(g["lam"] - c["lam"]) <= 1e-12 * max(1.0, abs(c["lam"]))
        for name in ("beta", "theta"):
            keys = set(g[name]) | set(c[name])
            for k in keys:
                assert abs(g[name].get(k, 0.0) - c[name].get(k, 0.0)) <= tol, (name, k, g[name].get(k), c[name].get(k))


@pytest.mark.parametrize("seed", [5, 6])
def test_dropin_lasso_path_matches_reference(seed):
    """xyz-regression (interaction Lasso) with the GPU screen: coefficients
    within 1e-4 of the all-CPU reference along the whole lambda path."""
    from paper_1610_05108_b200 import synth
    x, y, pairs, mains = synth.gauss(n=300, p=150, n_pairs=3, theta=1.0, noise_sd=0.5, n_mains=3, beta=1.0,
                                     seed=seed)
    kw = dict(grid_size=10, grid_ratio=0.05, kkt_l=50, kkt_max_candidates=16 * 150, seed=7, threads=1)
    cpu, _ = ck.lasso_path(ck.ref_lasso_lib(), x, y, **kw)
    gpu, _ = ck.lasso_path(ck.dropin_lib(), x, y, **kw)
    _compare_fits(gpu, cpu)
    # the path is non-trivial: mains and interaction terms enter it
    assert any(f["theta"] for f in gpu) and any(f["beta"] for f in gpu)


def _pm1_design(n, p, seed):
    from paper_1610_05108_b200.matrix import RealMatrix
    rng = np.random.default_rng(seed)
    xv = np.where(rng.random((p, n)) < 0.5, -1.0, 1.0)
    y = 1.5 * xv[2] + 1.2 * xv[5] * xv[9] - 1.0 * xv[11] * xv[40] + rng.normal(0.0, 0.4, n)
    return RealMatrix(xv), y


def test_dropin_lasso_binary_design_matches_reference():
    """+-1 design: square terms excluded, the KKT screen is the continuous-Y
    search on the packed matrix; the regression loop's scans on the GPU.
    Coefficients within 1e-4, the same active-set iteration counts."""
    x, y = _pm1_design(200, 120, 3)
    kw = dict(grid_size=8, grid_ratio=0.1, kkt_l=40, kkt_max_candidates=16 * 120, seed=5, threads=1)
    cpu, _ = ck.lasso_path(ck.ref_lasso_lib(), x, y, **kw)
    gpu, _ = ck.lasso_path(ck.dropin_lib(), x, y, **kw)
    _compare_fits(gpu, cpu)
    assert [f["iterations"] for f in gpu] == [f["iterations"] for f in cpu]
    assert [f["certified"] for f in gpu] == [f["certified"] for f in cpu]
    assert any(f["theta"] for f in gpu)


def test_dropin_lasso_large_p_matches_reference():
    """p = 2500 (no exhaustive certificate, probabilistic screens only):
    coefficients within 1e-4, iteration counts and degenerate flags equal,
    KKT residuals within 1e-9."""
    from paper_1610_05108_b200 import synth
    x, y, pairs, mains = synth.gauss(n=300, p=2500, n_pairs=3, theta=1.0, noise_sd=0.5, n_mains=4, beta=1.0, seed=8)
    kw = dict(grid_size=6, grid_ratio=0.2, kkt_l=60, kkt_max_candidates=16 * 2500, seed=7, threads=1)
    cpu, _ = ck.lasso_path(ck.ref_lasso_lib(), x, y, **kw)
    gpu, _ = ck.lasso_path(ck.dropin_lib(), x, y, **kw)
    _compare_fits(gpu, cpu)
    assert [f["iterations"] for f in gpu] == [f["iterations"] for f in cpu]
    assert [f["degenerate"] for f in gpu] == [f["degenerate"] for f in cpu]
    for g, c in zip(gpu, cpu):
        assert abs(g["kkt"] - c["kkt"]) <= 1e-9 * max(1.0, abs(c["kkt"]))


@pytest.mark.parametrize("design", ["gauss", "pm1"])
def test_dropin_kkt_check_interactions_matches_reference(design):
    """kkt_check_interactions (lasso.cpp:377-426) on the GPU: the same sorted
    violator lists as the reference at several lambda levels, including a
    level low enough that the screen degenerates to the exact all-pairs scan
    (p <= 2000)."""
    from paper_1610_05108_b200 import synth
    if design == "gauss":
        x, y, _, _ = synth.gauss(n=250, p=300, n_pairs=3, theta=1.0, noise_sd=0.5, n_mains=2, beta=1.0, seed=4)
    else:
        x, y = _pm1_design(250, 300, 4)
    r = np.asarray(y, np.float64) - np.mean(y)
    xc = x.values - x.values.mean(axis=1, keepdims=True)
    top = float(np.max(np.abs(np.triu((xc * r) @ xc.T, 1)))) / len(r)  # the strongest pair correlation
    seen_nonempty = False
    for frac in (1.2, 0.9, 0.6, 0.4) + ((1e-6,) if design == "pm1" else ()):  # pm1: means != 0 -> degenerate
        lam = top * frac
        kw = dict(kkt_l=60, kkt_max_candidates=0, seed=3, stream=2)  # unlimited (the reference default)
        want = ck.kkt_check_interactions(ck.ref_lasso_lib(), x, r, lam, **kw)
        got = ck.kkt_check_interactions(ck.dropin_lib(), x, r, lam, **kw)
        assert got == want, (design, frac)
        seen_nonempty |= bool(want)
    assert seen_nonempty


def test_design_correlations_vs_numpy():
    """xyzb_design_* (the regression loop's exact scans) against fp64 numpy:
    main correlations sum_i r_i (x_ij - m_j) and pair / square correlations
    sum_i r_i (x_ij - m_j)(x_ik - m_k), to 1e-12 of the sum of |terms|;
    out-of-range indices are data errors."""
    import ctypes as C
    from paper_1610_05108_b200 import _abi, _lib
    lib = _abi.bind(C.CDLL(_lib.LIB_PATH), _abi.SIGNATURES)
    rng = np.random.default_rng(9)
    n, p = 777, 1234
    xv = rng.normal(size=(p, n))  # column-major: column j is xv[j]
    means = xv.mean(axis=1)
    r = rng.normal(size=n)
    r -= r.mean()
    f64 = C.POINTER(C.c_double)
    d = C.c_void_p()
    err = _abi.errbuf()
    assert lib.xyzb_design_create(xv.ctypes.data_as(f64), n, p, means.ctypes.data_as(f64), 0, C.byref(d), err,
                                  _abi.ERRBUF) == 0, err.value
    try:
        out = np.zeros(p)
        assert lib.xyzb_design_main_correlations(d, r.ctypes.data_as(f64), out.ctypes.data_as(f64), err,
                                                 _abi.ERRBUF) == 0
        xc = xv - means[:, None]
        want = xc @ r
        assert np.all(np.abs(out - want) <= 1e-12 * (np.abs(xc) @ np.abs(r)))
        pairs = np.concatenate([rng.integers(0, p, (5000, 2)), np.repeat(np.arange(50), 2).reshape(-1, 2)])
        pairs = np.ascontiguousarray(pairs, np.uint32)
        pout = np.zeros(len(pairs))
        assert lib.xyzb_design_pair_correlations(d, r.ctypes.data_as(f64), pairs.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                 len(pairs), pout.ctypes.data_as(f64), err, _abi.ERRBUF) == 0
        terms = xc[pairs[:, 0]] * xc[pairs[:, 1]] * r
        assert np.all(np.abs(pout - terms.sum(axis=1)) <= 1e-12 * np.abs(terms).sum(axis=1))
        bad = np.array([0, p], np.uint32)
        assert lib.xyzb_design_pair_correlations(d, r.ctypes.data_as(f64), bad.ctypes.data_as(C.POINTER(C.c_uint32)),
                                                 1, pout.ctypes.data_as(f64), err, _abi.ERRBUF) == 3
    finally:
        lib.xyzb_design_destroy(d)


def test_dropin_unbiased_range_error_matches_reference():
    """Entries outside [-1, 1] with the unbiased transform: the same data_error
    (code 3, same message) from the drop-in (checked by the engine against the
    resident matrix) as from the reference (search.cpp:417-434)."""
    from paper_1610_05108_b200.matrix import RealMatrix
    from paper_1610_05108_b200.report import SearchConfig
    rng = np.random.default_rng(3)
    xv = rng.uniform(-1, 1, (40, 64))
    xv[7, 5] = 1.5
    x = RealMatrix(xv)
    y = rng.normal(size=64)
    cfg = SearchConfig(m=4, l=2, gamma=0.6, mode="continuous_xy", transform="unbiased")
    with pytest.raises(ck.CheckerError) as a:
        ck.ref_search(x, y, cfg)
    with pytest.raises(ck.CheckerError) as b:
        ck.dropin_search(x, y, cfg)
    assert a.value.code == b.value.code == 3
    assert str(a.value) == str(b.value)
    xv[7, 5] = 1.0  # in range again: the same pointer, new contents -> re-upload, no error
    ck.dropin_search(RealMatrix(xv), y, cfg)


def test_dropin_search_over_two_device_replicas(monkeypatch):
    """XYZ_GPU_DEVICES lists the GPUs the drop-in shards each search over (X
    replicated, repetitions split, shard results merged on the first): with
    two replicas on the test box's GPU the reference-facing xyz_search returns
    the reference's report."""
    monkeypatch.setenv("XYZ_GPU_DEVICES", "0,0")
    x = ck.ref_rademacher(700, 900, 12, 3)
    y = np.where(np.random.default_rng(6).random(700) < 0.5, 1, -1).astype(np.int8)
    from paper_1610_05108_b200.report import SearchConfig
    cfg = SearchConfig(m=7, l=9, gamma=0.57, seed=4, threads=1)
    got = ck.dropin_search(x, y, cfg)
    want = ck.ref_search(x, y, cfg)
    ok, msg = ck.same_hits(got, want)
    assert ok, msg
    assert (got.repetitions_run, got.candidates_enumerated, got.estimated_c) == \
        (want.repetitions_run, want.candidates_enumerated, want.estimated_c)


@pytest.mark.parametrize("mode", ["binary", "continuous_y", "sign", "unbiased"])
def test_dropin_sample_strengths_bit_exact_on_the_gpu(mode):
    """sample_strengths (search.cpp:229-291) in the drop-in draws its pairs on
    the host in the reference's RNG order and evaluates them on the GPU in the
    reference's order: every strength bit-identical, so optimal_m (the CLI's
    auto-M, xyz_main.cpp:142-167; the Lasso screen's M, lasso.cpp:184-192)
    picks the reference's M. Binary: Z = build_z(X, y) as the CLI builds it;
    unbiased: the Lasso's rescaled design (entries in [-1, 1])."""
    from paper_1610_05108_b200 import _abi
    rng = np.random.default_rng(3)
    n, p = 1000, 4000
    if mode in ("binary", "continuous_y"):
        x = ck.ref_rademacher(n, p, 21, 4)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8) if mode == "binary" else rng.standard_normal(n)
        if mode == "continuous_y":
            y[::17] = 0.0
        m, t = (_abi.MODE_BINARY if mode == "binary" else _abi.MODE_CONTINUOUS_Y), _abi.TRANSFORM_NONE
    else:
        g = ck.ref_gaussian(n, p, 5, 6)
        y = rng.standard_normal(n)
        if mode == "unbiased":
            x, y = ck.ref_rescale_rows(g, y)
        else:
            xv = g.values.copy()
            xv[rng.random(xv.shape) < 0.02] = 0.0
            from paper_1610_05108_b200 import RealMatrix
            x = RealMatrix(xv)
        m, t = _abi.MODE_CONTINUOUS_XY, (_abi.TRANSFORM_UNBIASED if mode == "unbiased" else _abi.TRANSFORM_SIGN)
    for count, gamma in ((2000, 0.506), (40000, 0.6)):
        want, want_m = ck.sample_strengths(ck.ref_lib(), x, y, m, t, count, gamma=gamma)
        got, got_m = ck.sample_strengths(ck.dropin_lib(), x, y, m, t, count, gamma=gamma)
        assert np.array_equal(got, want), (mode, count, np.max(np.abs(got - want)))
        assert got_m == want_m


def test_dropin_sample_strengths_errors_like_the_reference():
    from paper_1610_05108_b200 import _abi
    x = ck.ref_rademacher(100, 50, 1, 1)
    zero = np.zeros(100)
    for lib in (ck.ref_lib(), ck.dropin_lib()):
        with pytest.raises(ck.CheckerError, match="zero response vector"):
            ck.sample_strengths(lib, x, zero, _abi.MODE_CONTINUOUS_Y, _abi.TRANSFORM_NONE, 10)
        with pytest.raises(ck.CheckerError, match="need n_samples >= 1"):
            ck.sample_strengths(lib, x, np.ones(100), _abi.MODE_CONTINUOUS_Y, _abi.TRANSFORM_NONE, 0)
