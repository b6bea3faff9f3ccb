"""DRAM bytes per verified pair of a workload's verify kernel, for bench.py's
roofline (profiles/verify_traffic_<workload>.json).

  1. under ncu, one search of the workload (no timing):
       ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
           -k regex:verify_pairs --csv --log-file gpurun_out/vt.csv \
           python tools/verify_traffic.py run --config large --out gpurun_out/vt_run.json
  2. combine the per-launch DRAM bytes with the search's pair count:
       python tools/verify_traffic.py reduce --csv gpurun_out/vt.csv --run gpurun_out/vt_run.json \
           --out profiles/verify_traffic_large_cfg4.json
The search is deterministic (seeded data and draws), so the pair count of the
run under ncu is the count of every bench step.
"""
import argparse
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(args):
    import bench
    bench.select(args.config)
    import paper_1610_05108_b200 as xb
    x, y, _ = bench.make_data()
    cfg = bench.search_config(bench.WORKLOAD["l"])
    r = xb.Dataset(x).search(y, cfg)
    json.dump({"config": bench.WORKLOAD["name"], "verified_pairs": r.verified_pairs,
               "verify_launches": r.verify_launches, "verify_algorithmic_bytes": r.stage_bytes["verify"]},
              open(args.out, "w"))


def reduce(args):
    rows = [r for r in csv.reader(open(args.csv)) if len(r) > 5]
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), \
        hdr.index("Metric Unit")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
             "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0, "gpu__time_duration.sum": 0.0,
           "lts__t_bytes.sum": 0.0}
    launches = 0
    kernel = ""
    for r in rows[1:]:
        if "verify_pairs" not in r[ki] and "verify_binned" not in r[ki]:
            continue
        m = r[mi]
        if m in tot:
            tot[m] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
            if m == "gpu__time_duration.sum":
                launches += 1
                kernel = r[ki]
    rr = json.load(open(args.run))
    dram = tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]
    out = {"config": rr["config"], "kernel": kernel[:80], "launches": launches,
           "verified_pairs": rr["verified_pairs"], "dram_read_bytes": tot["dram__bytes_read.sum"],
           "dram_write_bytes": tot["dram__bytes_write.sum"], "dram_bytes_per_pair": dram / rr["verified_pairs"],
           "algorithmic_bytes_per_pair": rr["verify_algorithmic_bytes"] / rr["verified_pairs"],
           "ncu_ms": tot["gpu__time_duration.sum"] * 1e3,
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                     "--clock-control none over every verify launch of one search (tools/verify_traffic.py)"}
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("mode", choices=["run", "reduce"])
    ap.add_argument("--config", default="large")
    ap.add_argument("--csv")
    ap.add_argument("--run")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    run(a) if a.mode == "run" else reduce(a)
