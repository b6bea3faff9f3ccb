"""End-to-end throughput with several (X, y) jobs in flight (host threads):
every step a fresh Dataset from pinned host X (fp32 for real X, as bench.py's
e2e), search, results to host.
  python tools/e2e_pipeline.py large 1,2,3,4 [trace]
"""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import _lib  # noqa: E402

bench.select(sys.argv[1] if len(sys.argv) > 1 else "gwas")
flights = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "1,2,3,4").split(",")]
if len(sys.argv) > 3:
    _lib.set_test_option("trace", 1)
x, y, _ = bench.make_data()
cfg = bench.search_config(bench.WORKLOAD["l"])
src = x.words if hasattr(x, "words") else x.values.astype(np.float32)
pin = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True)
host = pin.numpy().view(src.dtype).reshape(src.shape)
host[...] = src
xh = xb.PackedMatrix(x.n_rows, x.n_cols, host) if hasattr(x, "words") else xb.RealMatrix(host, dtype=host.dtype)


def step(_=None):
    d = xb.Dataset(xh)
    r = d.search(y, cfg)
    d.close()
    return r


for nthreads in flights:
    with ThreadPoolExecutor(nthreads) as ex:
        list(ex.map(step, range(2 * nthreads)))
        torch.cuda.synchronize()
        n = max(4 * nthreads, 12)
        t0 = time.perf_counter()
        list(ex.map(step, range(n)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{nthreads} in flight: {1e3 * dt / n:.2f} ms/step, {n * 2 * bench.WORKLOAD['l'] / dt:.0f} runs/s", flush=True)
