"""Device time of one search per grouping path (config 2 data, several M)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import _lib, synth  # noqa: E402

x, y, _ = synth.gwas()
ds = xb.Dataset(x)
for m in [int(a) for a in (sys.argv[1:] or ["16", "17", "18", "19", "20"])]:
    for g in ("auto", "msplit", "part", "sort"):
        _lib.set_test_option("grouping", _lib.GROUPING[g])
        cfg = xb.SearchConfig(m=m, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False)
        try:
            for _ in range(2):
                ds.search(y, cfg)
            best = min(ds.search(y, cfg).device_ms for _ in range(3))
            r = ds.search(y, cfg)
            print(f"M={m} {g:7s} {best:7.3f} ms  sort {r.stage_ms['sort']:.3f} join {r.stage_ms['join']:.3f} "
                  f"verify {r.stage_ms['verify']:.3f} hits {len(r.hits)}", flush=True)
        except Exception as e:
            print(f"M={m} {g}: {e}", flush=True)
