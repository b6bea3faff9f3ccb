"""Where the end-to-end time of one search goes (host buffers in, results out).

Usage: python tools/e2e_breakdown.py [gwas|toy|cont|large] [pinned|pageable]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1610_05108_b200 as xb  # noqa: E402

config = sys.argv[1] if len(sys.argv) > 1 else "gwas"
mode = sys.argv[2] if len(sys.argv) > 2 else "pinned"
bench.select(config)
x, y, _ = bench.make_data()
cfg = bench.search_config(bench.WORKLOAD["l"])
src = x.words if hasattr(x, "words") else x.values
if mode == "pinned":
    pin = torch.empty(src.nbytes, dtype=torch.uint8, pin_memory=True)
    host = pin.numpy().view(src.dtype).reshape(src.shape)
    host[...] = src
    x = xb.PackedMatrix(x.n_rows, x.n_cols, host) if hasattr(x, "words") else xb.RealMatrix(host)
    dev = torch.empty(src.nbytes, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(pin, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"raw pinned H2D of X: {1e3 * dt:.2f} ms ({src.nbytes / dt / 1e9:.1f} GB/s)")
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
