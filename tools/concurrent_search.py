"""Device throughput of concurrent searches on resident datasets (config 2):
k host threads, one Dataset (stream) each, X already in HBM; wall clock over
all searches. Measures how much the search kernels of different streams
overlap (grouping is issue-bound, verify L2-bound)."""
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import torch

sys.path.insert(0, ".")
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402

x, y, _ = synth.gwas()
cfg = xb.SearchConfig(m=16, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False)
for k in (1, 2, 3, 4):
    ds = [xb.Dataset(x) for _ in range(k)]
    for d in ds:
        d.search(y, cfg)
    nper = 24 // k

    def work(d):
        for _ in range(nper):
            d.search(y, cfg)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with ThreadPoolExecutor(k) as ex:
        list(ex.map(work, ds))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{k} streams: {nper * k} searches in {dt * 1e3:.1f} ms -> {nper * k * 200 / dt:.0f} runs/s")
    for d in ds:
        d.close()
