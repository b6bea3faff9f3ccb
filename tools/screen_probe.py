"""One xyz-Lasso-like screen (config 5 data): continuous-XY unbiased search
at gamma ~ 0.5064, stage times."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402

L = bench.LASSO
x, y, pairs, mains = synth.gauss(L["n"], L["p"], L["n_pairs"], L["theta"], L["noise_sd"], L["n_mains"], L["beta"],
                                 L["seed"])
from tests import checkers as ck  # noqa: E402

xr, yr = ck.ref_rescale_rows(x, y)  # lasso.cpp:129-139: X / nu (entries in [-1, 1]), y * nu^2
ds = xb.Dataset(xr)
y = yr
for m in (int(a) for a in (sys.argv[1:] or ["8", "12", "16"])):
    cfg = xb.SearchConfig(m=m, l=100, gamma=0.5064, seed=7, mode="continuous_xy", transform="unbiased",
                          max_candidates_per_rep=16 * L["p"], estimate_complexity=False)
    ds.search(y, cfg)
    r = ds.search(y, cfg)
    print(f"M={m}: {r.device_ms:.2f} ms, hits {len(r.hits)}, aborted {r.aborted_repetitions}/{r.repetitions_run}, "
          f"verified {r.verified_pairs}, stages " + " ".join(f"{k}={v:.2f}" for k, v in r.stage_ms.items() if v),
          flush=True)
