"""Measurement (round 2): config 4's binned verify under z-window sizes
(engine test option binned_wshift); device time of one search, best of 3, the
verify and join stages, and the top-K against the first setting's.
  python tools/binned_sweep.py 15,16,17 [option] [config]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1610_05108_b200 import _lib  # noqa: E402

bench.select(sys.argv[3] if len(sys.argv) > 3 else "large")
import paper_1610_05108_b200 as xb  # noqa: E402

x, y, _ = bench.make_data()
cfg = bench.search_config(bench.WORKLOAD["l"])
ds = xb.Dataset(x)
ds.search(y, cfg)
ref = None
opt = sys.argv[2] if len(sys.argv) > 2 else "binned_wshift"
for ws in [int(a) for a in sys.argv[1].split(",")]:
    _lib.set_test_option(opt, ws)
    best = None
    for _ in range(3):
        r = ds.search(y, cfg)
        if best is None or r.device_ms < best.device_ms:
            best = r
    key = [(h.j, h.k, h.strength, h.found_at_repetition) for h in best.top_hits()]
    ref = ref or key
    print(f"{opt} {ws}: {best.device_ms:.2f} ms  verify {best.stage_ms['verify']:.2f}  "
          f"join {best.stage_ms['join']:.2f}  same top-K {key == ref}", flush=True)
