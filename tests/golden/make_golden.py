"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Runs the unmodified reference core (oracle/_ref/libxyzref.so, built from
/root/reference by `make -C oracle`) on small seeded cases that mirror the
reference's own tests for this path (proj/tests/test_pair_search.cpp,
test_search.cpp, test_projection.cpp, test_packed_matrix.cpp,
acceptance_main.cpp) plus BASELINE config 1 at full size, and stores inputs
and outputs as .npz. Re-run with:  python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1610_05108_b200.matrix import PackedMatrix, RealMatrix  # noqa: E402
from paper_1610_05108_b200.report import SearchConfig  # noqa: E402
from tests import checkers as ck  # noqa: E402


def hits_arrays(rep, prefix="hits"):
    a = rep.hit_array()
    return {
        f"{prefix}_j": a["j"], f"{prefix}_k": a["k"], f"{prefix}_strength": a["strength"],
        f"{prefix}_rep": a["rep"], f"{prefix}_sign": a["sign"],
        "repetitions_run": np.uint64(rep.repetitions_run),
        "aborted_repetitions": np.uint64(rep.aborted_repetitions),
        "candidates_enumerated": np.uint64(rep.candidates_enumerated),
        "candidates_checked": np.uint64(rep.candidates_checked),
        "estimated_c": np.float64(rep.estimated_c),
        "gamma0": np.float64(rep.gamma0),
        "top_k": np.array(rep.top_k, np.uint64),
    }


def cfg_arrays(cfg: SearchConfig):
    return {
        "cfg_m": np.uint64(cfg.m), "cfg_l": np.uint64(cfg.l), "cfg_gamma": np.float64(cfg.gamma),
        "cfg_mode": np.array(cfg.mode), "cfg_transform": np.array(cfg.transform),
        "cfg_negatives": np.bool_(cfg.search_negatives), "cfg_seed": np.uint64(cfg.seed),
        "cfg_guard": np.uint64(cfg.max_candidates_per_rep), "cfg_stop": np.bool_(cfg.stop_after_first_hit),
        "cfg_estimate": np.bool_(cfg.estimate_complexity), "cfg_sample": np.uint64(cfg.strength_sample_size),
        "cfg_top_k": np.uint64(cfg.top_k),
    }


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)


def search_case(name, x, y, cfg):
    cfg.threads = 1  # candidates_checked is thread-dependent in the reference; fixtures pin threads=1
    rep = ck.ref_search(x, y, cfg)
    arrays = dict(cfg_arrays(cfg), **hits_arrays(rep))
    if isinstance(x, PackedMatrix):
        arrays.update(x_words=x.words, n=np.uint64(x.n_rows), p=np.uint64(x.n_cols))
    else:
        arrays.update(x_real=x.values, n=np.uint64(x.n_rows), p=np.uint64(x.n_cols))
    arrays["y"] = np.asarray(y)
    save(name, **arrays)
    return rep


def main():
    cases = []
    # --- equal_pairs: the paper's Fig. 2 configuration (test_pair_search.cpp:37-54) ---
    xv = np.array([10, 20, 30, 40, 50, 60, 70, 80, 70], np.uint64)
    zv = np.array([70, 50, 110, 30, 70, 30, 120, 130, 140], np.uint64)
    pairs, total = ck.ref_equal_pairs(xv, zv)
    save("equal_pairs_fig2", x_keys=xv, z_keys=zv, pairs=pairs, total=np.uint64(total))
    # random equal_pairs (test_pair_search.cpp:72-90 shape)
    rng = np.random.default_rng(31)
    ex = {}
    for t in range(20):
        p = int(rng.integers(1, 65))
        alpha = int(rng.integers(1, 9))
        a = rng.integers(0, alpha, p).astype(np.uint64)
        b = rng.integers(0, alpha, p).astype(np.uint64)
        pr, tot = ck.ref_equal_pairs(a, b)
        ex[f"x{t}"], ex[f"z{t}"], ex[f"pairs{t}"], ex[f"total{t}"] = a, b, pr, np.uint64(tot)
    save("equal_pairs_random", count=np.uint64(20), **ex)

    # --- draws + project_keys (test_projection.cpp:49-102) ---
    x = ck.ref_rademacher(200, 37, 3, 0)
    d = {}
    for t, (seed, stream, m) in enumerate([(3, 1, 8), (3, 2, 16), (7, 11, 23), (9, 5, 64), (1, 1, 1)]):
        draw = ck.ref_draw_subsample(200, m, seed, stream)
        d[f"draw{t}"] = draw
        d[f"keys{t}"] = ck.ref_project_keys(x, draw)
        d[f"seed{t}"], d[f"stream{t}"], d[f"m{t}"] = np.uint64(seed), np.uint64(stream), np.uint64(m)
    yw = np.random.default_rng(5).normal(size=200)
    yw[:7] = 0.0
    d["y_weighted"] = yw
    d["draw_weighted"] = ck.ref_draw_subsample(200, 20, 4, 9, yw)
    save("projection", x_words=x.words, n=np.uint64(200), p=np.uint64(37), count=np.uint64(5), **d)

    # --- binary searches mirroring test_search.cpp ---
    x, y = ck.ref_planted(64, 12, 0, 1, 1.0, 7)
    search_case("bin_perfect", x, y, SearchConfig(m=9, l=1, gamma=1.0, seed=123, top_k=5))
    x, y = ck.ref_planted(128, 48, 0, 1, 0.85, 3)
    search_case("bin_threads", x, y, SearchConfig(m=4, l=16, gamma=0.7, seed=77, estimate_complexity=False, threads=1,
                                                  top_k=20))
    x = ck.ref_rademacher(96, 40, 31, 5)
    yy = np.where(np.random.default_rng(96).random(96) < 0.5, 1, -1).astype(np.int8)
    search_case("bin_oracle_check", x, yy, SearchConfig(m=2, l=10, gamma=0.55, seed=9, threads=1,
                                                        strength_sample_size=2000, top_k=50))
    x, y = ck.ref_planted(64, 10, 0, 1, 0.0, 13)
    search_case("bin_negated", x, y, SearchConfig(m=6, l=2, gamma=1.0, seed=4, threads=1))
    # guard: all columns equal (test_search.cpp:333-354)
    n, p = 64, 32
    g = np.random.default_rng(51)
    rows = np.where(g.random(n) < 0.5, 1, -1).astype(np.int8)
    x = PackedMatrix.from_signs(np.repeat(rows[:, None], p, axis=1))
    search_case("bin_guard", x, np.ones(n, np.int8), SearchConfig(m=8, l=3, gamma=0.9, search_negatives=False,
                                                                  max_candidates_per_rep=10, seed=5, threads=1))
    # stop_after_first_hit
    x, y = ck.ref_planted(200, 80, 3, 9, 0.95, 17)
    search_case("bin_stop_first", x, y, SearchConfig(m=5, l=12, gamma=0.9, seed=11, stop_after_first_hit=True,
                                                     estimate_complexity=False))
    # sweep: n straddling word boundaries, guard on/off, M variety (Appendix A "Validated")
    k = 0
    for n in (63, 64, 65, 200):
        for m, guard in ((4, 0), (6, 150), (3, 0)):
            x = ck.ref_rademacher(n, 300, 100 + k, 1)
            yy = np.where(np.random.default_rng(k).random(n) < 0.5, 1, -1).astype(np.int8)
            search_case(f"bin_sweep{k:02d}", x, yy, SearchConfig(m=m, l=5, gamma=0.6, seed=k + 7,
                                                                 max_candidates_per_rep=guard, threads=1,
                                                                 strength_sample_size=500, top_k=10))
            k += 1
    # BASELINE config 1 at full size: toy 1000 x 2000, M=8, L=10, gamma 0.55, seed 7, K=10
    x, y = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    rep = search_case("cfg1_toy", x, y, SearchConfig(m=8, l=10, gamma=0.55, seed=7, threads=1, top_k=10))
    print("cfg1 hits", len(rep.hits), "enumerated", rep.candidates_enumerated)

    # --- continuous-Y (test_search.cpp:356-376) ---
    x = ck.ref_rademacher(200, 16, 61, 0)
    s = x.to_signs()
    u = np.random.default_rng(61).random(200)
    yc = s[:, 0].astype(float) * s[:, 1] * (0.5 + u)
    search_case("cy_planted", x, yc, SearchConfig(m=6, l=3, gamma=0.99, seed=8, mode="continuous_y", top_k=3))
    for t in range(3):
        x = ck.ref_rademacher(150, 120, 200 + t, 2)
        yc = np.random.default_rng(t).normal(size=150)
        yc[np.random.default_rng(t + 9).random(150) < 0.1] = 0.0
        search_case(f"cy_random{t}", x, yc, SearchConfig(m=4, l=6, gamma=0.56, seed=t, mode="continuous_y",
                                                         threads=1, strength_sample_size=400, top_k=15))

    # --- continuous-XY (test_search.cpp:378-432) ---
    xr = ck.ref_uniform(2000, 6, 71, 0)
    yr = xr.values[0] * xr.values[1]
    search_case("cxy_unbiased_planted", xr, yr, SearchConfig(m=2, l=12, gamma=0.70, seed=15, search_negatives=False,
                                                             mode="continuous_xy", transform="unbiased"))
    xg = ck.ref_gaussian(500, 8, 81, 0)
    sg = np.sign(xg.values)
    yg = sg[0] * sg[1] * (0.2 + np.random.default_rng(81).random(500))
    search_case("cxy_sign_planted", xg, yg, SearchConfig(m=4, l=2, gamma=0.999, seed=30, search_negatives=False,
                                                         mode="continuous_xy", transform="sign"))
    for t, tr in enumerate(("sign", "unbiased", "sign", "unbiased")):
        xr = ck.ref_uniform(180, 90, 300 + t, 3)
        v = xr.values.copy()
        if t >= 2:
            v[np.random.default_rng(t).random(v.shape) < 0.1] = 0.0  # exact zeros: coin path
        xr = RealMatrix(v)
        yr = np.random.default_rng(t + 50).normal(size=180)
        search_case(f"cxy_random{t}", xr, yr, SearchConfig(m=3, l=5, gamma=0.55, seed=t + 3, mode="continuous_xy",
                                                           transform=tr, threads=1, strength_sample_size=300,
                                                           top_k=25))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
