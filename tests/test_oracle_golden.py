"""Pin the CPU restatement (oracle/liboracle.so) to the reference's own outputs.

The golden fixtures were produced by the unmodified reference core
(tests/golden/make_golden.py). A restatement that differs from them in any
field is not a valid checker for the GPU engine.
"""
import os

import numpy as np
import pytest

from tests.helpers import GOLDEN, expected_hits, golden_names, load_case, report_hits
from tests import checkers as ck

SEARCH_CASES = [n for n in golden_names() if n.split("_")[0] in ("bin", "cfg1", "cy", "cxy")]


@pytest.mark.parametrize("name", SEARCH_CASES)
def test_oracle_matches_reference_fixture(name):
    x, y, cfg, z = load_case(name)
    rep = ck.oracle_search(x, y, cfg)
    assert report_hits(rep) == expected_hits(z)  # bit-exact, including fp64 strengths
    assert rep.repetitions_run == int(z["repetitions_run"])
    assert rep.aborted_repetitions == int(z["aborted_repetitions"])
    assert rep.candidates_enumerated == int(z["candidates_enumerated"])
    assert rep.candidates_checked == int(z["candidates_checked"])  # threads=1 semantics
    assert rep.estimated_c == float(z["estimated_c"])
    assert rep.gamma0 == float(z["gamma0"])
    assert rep.top_k == z["top_k"].tolist()


def test_oracle_equal_pairs_fig2():
    z = np.load(os.path.join(GOLDEN, "equal_pairs_fig2.npz"))
    pairs, total = ck.oracle_equal_pairs(z["x_keys"], z["z_keys"])
    assert total == int(z["total"]) == 7
    assert pairs.tolist() == z["pairs"].tolist()
    # the paper's 1-based picture: {3}x{4,6} u {5}x{2} u {7,9}x{1,5}
    assert sorted(map(tuple, pairs.tolist())) == sorted([(2, 3), (2, 5), (4, 1), (6, 0), (6, 4), (8, 0), (8, 4)])


def test_oracle_equal_pairs_random():
    z = np.load(os.path.join(GOLDEN, "equal_pairs_random.npz"))
    for t in range(int(z["count"])):
        pairs, total = ck.oracle_equal_pairs(z[f"x{t}"], z[f"z{t}"])
        assert total == int(z[f"total{t}"])
        assert pairs.tolist() == z[f"pairs{t}"].tolist()


def test_oracle_project_keys_and_draws():
    from paper_1610_05108_b200.matrix import PackedMatrix

    z = np.load(os.path.join(GOLDEN, "projection.npz"))
    x = PackedMatrix(int(z["n"]), int(z["p"]), z["x_words"])
    for t in range(int(z["count"])):
        draw = z[f"draw{t}"].astype(np.uint32)
        keys = ck.oracle_project_keys(x, draw[None, :])[0]
        assert keys.tolist() == z[f"keys{t}"].tolist()
    # draws: oracle_draws(L=stream) reproduces draw_subsample on make_stream(seed, stream)
    for t in range(int(z["count"])):
        seed, stream, m = int(z[f"seed{t}"]), int(z[f"stream{t}"]), int(z[f"m{t}"])
        d = ck.oracle_draws(int(z["n"]), m, stream, False, seed)
        assert d[0, stream - 1].tolist() == z[f"draw{t}"].tolist()
    d = ck.oracle_draws(int(z["n"]), 20, 9, False, 4, z["y_weighted"])
    assert d[0, 8].tolist() == z["draw_weighted"].tolist()
    assert not np.isin(np.arange(7), d).any()  # zero-weight rows are never drawn


@pytest.mark.skipif(not ck.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_random():
    """Randomised equivalence against the live reference (Appendix A 'Validated')."""
    rng = np.random.default_rng(2024)
    for t in range(12):
        n = int(rng.choice([63, 64, 65, 130]))
        p = int(rng.integers(20, 200))
        x = ck.ref_rademacher(n, p, 500 + t, 4)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        from paper_1610_05108_b200.report import SearchConfig
        cfg = SearchConfig(m=int(rng.integers(1, 7)), l=4, gamma=float(rng.choice([0.55, 0.6, 0.7])), seed=t,
                           max_candidates_per_rep=int(rng.choice([0, 60])), threads=1, strength_sample_size=300,
                           top_k=7)
        a, b = ck.ref_search(x, y, cfg), ck.oracle_search(x, y, cfg)
        ok, msg = ck.same_hits(a, b)
        assert ok, msg
        assert (a.candidates_enumerated, a.aborted_repetitions, a.candidates_checked, a.estimated_c, a.top_k) == \
               (b.candidates_enumerated, b.aborted_repetitions, b.candidates_checked, b.estimated_c, b.top_k)
