"""Continuous-Y (weighted, A9) search on a +-1 design, the Lasso screen's
shape (n=1000, p=20000, M=12, L=100, real response): device and verify time
of the bit-plane pair verify against the exact set-bit-sum item walk."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import _lib, synth  # noqa: E402

x, _ = synth.toy(1000, 20000, 4, 16, 0.9, 5)
y = np.random.default_rng(5).standard_normal(1000)
ds = xb.Dataset(x)
for label, off in (("bit planes, pair list", 0), ("exact sums, item walk", 1)):
    _lib.set_test_option("sign_verify_off", off)
    cfg = xb.SearchConfig(m=12, l=100, gamma=0.55, seed=7, top_k=100, mode="continuous_y", estimate_complexity=False)
    ds.search(y, cfg)
    r = min((ds.search(y, cfg) for _ in range(5)), key=lambda r: r.device_ms)
    print(f"{label:24s} device {r.device_ms:7.3f} ms  verify {r.stage_ms['verify']:7.3f} ms  "
          f"pairs {r.verified_pairs}  hits {len(r.hits)}  runs/s {r.runs_executed / r.device_ms * 1e3:.0f}", flush=True)
_lib.set_test_option("sign_verify_off", 0)
