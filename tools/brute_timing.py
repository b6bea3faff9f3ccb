"""Time the GPU exhaustive oracle at BASELINE config 2 size and the
reference's brute force on a bounded sample (pairs/s)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402

x, y, _ = synth.gwas()
ds = xb.Dataset(x)
p = x.n_cols
for opt in (dict(histogram_bins=100), dict(top_k=100), dict(gamma=0.6)):
    xb.brute_force_search(ds, y, force=True, **opt)
    t0 = time.perf_counter()
    r = xb.brute_force_search(ds, y, force=True, **opt)
    dt = time.perf_counter() - t0
    print(f"GPU brute force p={p} n={x.n_rows} {opt}: {dt * 1e3:.1f} ms, {r.pairs_scanned / dt:.3e} pairs/s, "
          f"{len(r.pairs)} pairs", flush=True)
try:
    from tests import checkers as ck
    sub = xb.PackedMatrix(x.n_rows, 600, x.words[:600].copy())
    t0 = time.perf_counter()
    pairs, scanned, _ = ck.ref_brute_force(sub, y, top_k=100, force=True)
    dt = time.perf_counter() - t0
    print(f"reference brute force p=600 n={x.n_rows} top_k=100: {dt:.2f} s, {scanned / dt:.3e} pairs/s", flush=True)
except Exception as e:  # the reference core is not built on this host
    print("reference brute force unavailable:", e)
