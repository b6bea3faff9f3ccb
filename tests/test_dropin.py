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
