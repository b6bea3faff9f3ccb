"""Shared helpers of the test suite (fixture loading, hit-list views)."""
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_names(prefix=""):
    return sorted(f[:-4] for f in os.listdir(GOLDEN) if f.endswith(".npz") and f.startswith(prefix))


def load_case(name):
    """(x, y, cfg, expected) from a golden search fixture."""
    from paper_1610_05108_b200.matrix import PackedMatrix, RealMatrix
    from paper_1610_05108_b200.report import SearchConfig

    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    n, p = int(z["n"]), int(z["p"])
    x = PackedMatrix(n, p, z["x_words"]) if "x_words" in z else RealMatrix(z["x_real"])
    cfg = SearchConfig(m=int(z["cfg_m"]), l=int(z["cfg_l"]), gamma=float(z["cfg_gamma"]), mode=str(z["cfg_mode"]),
                       transform=str(z["cfg_transform"]), search_negatives=bool(z["cfg_negatives"]),
                       seed=int(z["cfg_seed"]), max_candidates_per_rep=int(z["cfg_guard"]),
                       stop_after_first_hit=bool(z["cfg_stop"]), estimate_complexity=bool(z["cfg_estimate"]),
                       strength_sample_size=int(z["cfg_sample"]), top_k=int(z["cfg_top_k"]), threads=1)
    return x, z["y"], cfg, z


def expected_hits(z):
    return list(zip(z["hits_j"].tolist(), z["hits_k"].tolist(), z["hits_strength"].tolist(), z["hits_rep"].tolist(),
                    z["hits_sign"].tolist()))


def report_hits(rep):
    return [(h.j, h.k, h.strength, h.found_at_repetition, h.sign) for h in rep.hits]
