"""Measure verify-kernel variants on one dataset (env knobs read per search)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "gwas"
bench.select(config)
x, y, _ = bench.make_data()
ds = xb.Dataset(x)
cfg = bench.search_config(bench.WORKLOAD["l"])
variants = [("simple", "4"), ("simple", "2"), ("simple", "1"), ("pipelined", "4"), ("pipelined", "2"),
            ("pipelined", "1")]
out = {}
for v, ch in variants:
    os.environ["XYZB_VERIFY"] = v
    os.environ["XYZB_VP_CHUNKS"] = ch
    for _ in range(2):
        ds.search(y, cfg)
    vs, tot = [], []
    for _ in range(5):
        r = ds.search(y, cfg)
        vs.append(r.verify_kernel_ms)
        tot.append(r.device_ms)
    out[f"{v}/{ch}"] = (min(vs), min(tot), len(r.hits))
    print(v, ch, "verify ms", round(min(vs), 3), "search ms", round(min(tot), 3), "hits", len(r.hits), flush=True)
json.dump(out, open(os.path.join("gpurun_out", f"sweep_{config}.json"), "w"), indent=1)
