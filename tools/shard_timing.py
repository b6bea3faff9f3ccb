"""Measurement (round 2): strong scaling of a search, one shard at a time on ONE
GPU. The runs of each pass split into contiguous shards exactly as
parallel.shard_config / xyzb_problem.devices split them over N GPUs; a shard
shares nothing with the others until the exchange (a few KB of top-K hits),
so the device time of the slowest shard is what an N-GPU step takes before
that exchange. This is NOT a multi-GPU measurement: the all-gather and merge
(exchange_ms_per_step in bench.py --gpus N) are not in it.
  python tools/shard_timing.py [config] [1,2,4,8]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

bench.select(sys.argv[1] if len(sys.argv) > 1 else "large")
import paper_1610_05108_b200 as xb  # noqa: E402
from paper_1610_05108_b200 import parallel  # noqa: E402

worlds = [int(a) for a in (sys.argv[2] if len(sys.argv) > 2 else "1,2,4,8").split(",")]
x, y, _ = bench.make_data()
L = bench.WORKLOAD["l"]
cfg = bench.search_config(L)
ds = xb.Dataset(x)
ds.search(y, cfg)
passes = 2 if cfg.search_negatives else 1
base = None
out = []
for world in worlds:
    worst = None
    for rank in sorted({0, world // 2, world - 1}):
        c = parallel.shard_config(cfg, rank, world)
        ds.search(y, c)  # capacities settle on the shard's fills
        best = min((ds.search(y, c) for _ in range(3)), key=lambda r: r.device_ms)
        if worst is None or best.device_ms > worst.device_ms:
            worst = best
    runs_s = passes * L / (worst.device_ms * 1e-3)
    base = base or runs_s
    row = {"shards": world, "runs_per_shard": worst.repetitions_run, "slowest_shard_ms": round(worst.device_ms, 3),
           "runs_per_s_all_shards": round(runs_s, 1), "vs_one_shard": round(runs_s / base, 3),
           "efficiency": round(runs_s / base / world * worlds[0], 3),
           "stage_ms": {k: round(v, 3) for k, v in worst.stage_ms.items()}}
    out.append(row)
    print(json.dumps(row), flush=True)
