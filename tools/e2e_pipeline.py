"""End-to-end throughput with several (X, y) jobs in flight (host threads)."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402

bench.select(sys.argv[1] if len(sys.argv) > 1 else "gwas")
x, y, _ = bench.make_data()
cfg = bench.search_config(bench.WORKLOAD["l"])
pin = torch.empty(x.words.nbytes, dtype=torch.uint8, pin_memory=True)
host = pin.numpy().view(x.words.dtype).reshape(x.words.shape)
host[...] = x.words
xh = xb.PackedMatrix(x.n_rows, x.n_cols, host)


def step(_=None):
    d = xb.Dataset(xh)
    r = d.search(y, cfg)
    d.close()
    return r


for nthreads in (1, 2, 3, 4):
    with ThreadPoolExecutor(nthreads) as ex:
        list(ex.map(step, range(2 * nthreads)))
        torch.cuda.synchronize()
        n = 24
        t0 = time.perf_counter()
        list(ex.map(step, range(n)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{nthreads} in flight: {1e3 * dt / n:.2f} ms/step, {n * 2 * bench.WORKLOAD['l'] / dt:.0f} runs/s", flush=True)
