"""BASELINE config 5 with the reference's default kkt_max_candidates = 0
(no guard): the all-CPU reference runs out of host memory;
through the drop-in the screen's candidates stay on the device."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402
from tests import checkers as ck  # noqa: E402

L = bench.LASSO
x, y, pairs, mains = synth.gauss(L["n"], L["p"], L["n_pairs"], L["theta"], L["noise_sd"], L["n_mains"], L["beta"],
                                 L["seed"])
grid = int(sys.argv[1]) if len(sys.argv) > 1 else L["grid_size"]
kw = dict(grid_size=grid, grid_ratio=L["grid_ratio"], kkt_l=L["kkt_l"], kkt_max_candidates=0, seed=L["path_seed"])
t0 = time.perf_counter()
fits, w = ck.lasso_path(ck.dropin_lib(), x, y, threads=1, **kw)
print(f"drop-in lasso, kkt_max_candidates=0 (unguarded), {grid} lambdas: {w:.2f} s, {len(fits)} fits, "
      f"final support {len(fits[-1]['beta'])} mains / {len(fits[-1]['theta'])} pairs", flush=True)
