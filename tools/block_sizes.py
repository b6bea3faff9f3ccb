"""How the canonical candidates of a config 2 search split by block size
(hc x sc pairs of key v and its partner v ^ c): the share a tiled verify of
large blocks could read once per column instead of once per pair."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402
from tests import checkers as ck  # noqa: E402

x, y, _ = synth.gwas()
n, p, M, L = x.n_rows, x.n_cols, 16, 100
draws = ck.oracle_draws(n, M, L, True, 7).reshape(2 * L, M)  # pass-major rows
ds = xb.Dataset(x)
keys = ds.project_keys(draws)
tot = {"<=32": 0, "33-1024": 0, ">1024": 0}
cols_read = {"pairs": 0, "tiles": 0}
minside = {1: 0, 2: 0, 3: 0, 4: 0, 8: 0}  # pairs of blocks > 32 pairs by their smaller side (>= key)
for r in range(draws.shape[0]):
    rows = draws[r]
    ybits = (y[rows] > 0).astype(np.uint64)
    yk = int(sum(int(b) << s for s, b in enumerate(ybits)))
    mask = (1 << M) - 1
    c = (~yk & mask) if r < L else yk
    cnt = np.bincount(keys[r].astype(np.int64), minlength=1 << M)
    v = np.arange(1 << M)
    v2 = v ^ c
    sel = v2 > v if c else v2 == v
    a, b = cnt[v[sel]], cnt[v2[sel]]
    work = a * b if c else a * (a - 1) // 2
    for lo, hi, k in ((0, 32, "<=32"), (33, 1024, "33-1024"), (1025, 1 << 62, ">1024")):
        m = (work >= lo) & (work <= hi)
        tot[k] += int(work[m].sum())
    big = work > 32
    small_side = np.minimum(a, b) if c else a
    for k in sorted(minside, reverse=True):
        m = big & (small_side >= k)
        minside[k] += int(work[m].sum())
        big_rest = big & (small_side < k)
    cols_read["pairs"] += int(2 * work.sum())
    cols_read["tiles"] += int(2 * work[~big].sum() + (a[big] + b[big]).sum())
print("canonical pairs by block size:", tot, "total", sum(tot.values()))
print("columns read: one per pair side", cols_read["pairs"], "| large blocks as tiles", cols_read["tiles"])
print("pairs of >32-pair blocks whose smaller side is >= k columns:", minside)
