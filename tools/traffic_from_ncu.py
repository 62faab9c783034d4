"""ncu launch list (CSV, gpu__time_duration + dram bytes) -> profiles/traffic.json.

Per kernel: launches, average DRAM bytes (read + write) per launch and average
cold/serialized duration. bench.py reads this file to fill roofline.traffic
for the dominant kernel (the bytes a real launch moved, against the
algorithmic bytes it reports as `achieved`).
Usage: python tools/traffic_from_ncu.py gpurun_out/prof_round/launches.csv profiles/traffic.json <label> [workload]
"""
import csv
import json
import sys
from collections import defaultdict

UNIT = {"byte": 1.0, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9,
        "nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}


def main(src, dst, label, workload="caltech256"):
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui, idi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    agg = defaultdict(lambda: defaultdict(float))
    ids = defaultdict(set)
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        raw = r[ki].split("(")[0].replace("void ", "").replace("ddcca::", "")
        name = raw.split("<")[0]
        if name == "conv_hist_tc_kernel" and ("true" in raw or raw.endswith(", 1>")):
            name = "conv_resp_tc_kernel"  # the responses mode of the tensor-core conv (hidden layers)
        if name == "lag_tma_kernel" and ("true" in raw or raw.endswith(", 1>")):
            name = "lag_tma_blk_kernel"  # the blocked (float32-product) instantiation
        agg[name][r[mi]] += float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        ids[name].add(r[idi])
    out = {"source": label, "workload": workload, "kernels": {}}
    for name, a in agg.items():
        n = len(ids[name])
        out["kernels"][name] = {
            "launches": n,
            "dram_bytes_per_launch": (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / n,
            "ms_per_launch_cold": a["gpu__time_duration.sum"] / n,
        }
    json.dump(out, open(dst, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main(*sys.argv[1:5])
