"""Where the end-to-end time of one search goes (host buffers in, results out)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "gwas"
bench.select(config)
x, y, _ = bench.make_data()
cfg = bench.search_config(bench.WORKLOAD["l"])
for it in range(4):
    t0 = time.perf_counter()
    ds = xb.Dataset(x)
    t1 = time.perf_counter()
    rep = ds.search(y, cfg)
    t2 = time.perf_counter()
    ds.close()
    t3 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.2f} ms  search {1e3*(t2-t1):.2f} ms (device {rep.device_ms:.2f})  "
          f"destroy {1e3*(t3-t2):.2f} ms  total {1e3*(t3-t0):.2f} ms", flush=True)
