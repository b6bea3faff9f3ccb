"""Concurrency probe: several host threads searching their own datasets
(own streams) — does the engine overlap them? Prints wall time per step for
1 and 4 threads, with and without dataset creation, per top-K mode."""
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import synth  # noqa: E402

x, y, _ = synth.gwas()
pin = torch.empty(x.words.nbytes, dtype=torch.uint8, pin_memory=True)
pw = pin.numpy().view(x.words.dtype).reshape(x.words.shape)
pw[...] = x.words
xh = xb.PackedMatrix(x.n_rows, x.n_cols, pw)
for mode in ("hits", "candidates"):
    cfg = xb.SearchConfig(m=16, l=100, gamma=0.6, seed=7, top_k=100, estimate_complexity=False, top_k_mode=mode)
    dss = [xb.Dataset(xh) for _ in range(4)]
    for d in dss:
        d.search(y, cfg)
    for nthr in (1, 4):
        with ThreadPoolExecutor(nthr) as ex:
            list(ex.map(lambda i: dss[i % 4].search(y, cfg), range(8)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            list(ex.map(lambda i: dss[i % 4].search(y, cfg), range(32)))
            torch.cuda.synchronize()
            print(f"{mode:10s} search only, {nthr} threads: {1e3 * (time.perf_counter() - t0) / 32:.3f} ms/step",
                  flush=True)

            def step(i):
                d = xb.Dataset(xh)
                r = d.search(y, cfg)
                d.close()
                return r
            list(ex.map(step, range(8)))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            list(ex.map(step, range(32)))
            torch.cuda.synchronize()
            print(f"{mode:10s} create+search, {nthr} threads: {1e3 * (time.perf_counter() - t0) / 32:.3f} ms/step",
                  flush=True)
