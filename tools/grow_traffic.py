"""DRAM traffic of the wide grower from an ncu metrics capture of one fit.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --csv --log-file t.csv python tools/fit_once.py c4 148
    python tools/grow_traffic.py t.csv TREES SPLIT_ROWS N MTRY > profiles/x.json

Sums per kernel; reports measured DRAM bytes per tree next to the SURVEY 8d algorithmic
bytes per tree, B_tree = 4n + split_rows/T * (24*mtry + 16).
"""
import collections
import csv
import json
import sys

rows = list(csv.reader(open(sys.argv[1])))
T, split_rows, n, mtry = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ik, iid, im, iu, iv = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Unit",
                                            "Metric Value"))
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
        "nsecond": 1e-6, "usecond": 1e-3,
        "msecond": 1.0}
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[start + 1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0].replace("void ", "").replace("aiwc_b200::", "")
    v = float(r[iv].replace(",", "")) * unit.get(r[iu], 1.0)
    per[k][r[im]] += v
    per[k]["launches"] += 1 if r[im] == "gpu__time_duration.sum" else 0
tot_b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in per.values())
tot_ms = sum(d["gpu__time_duration.sum"] for d in per.values())
alg = 4 * n * T + split_rows * (24 * mtry + 16)
out = {"trees": T, "split_rows": split_rows, "dram_bytes": tot_b, "dram_bytes_per_tree": tot_b / T,
       "algorithmic_bytes_per_tree": alg / T, "traffic_over_algorithmic": tot_b / alg,
       "kernel_ms_serialised": tot_ms,
       "kernels": {k: {"launches": int(d["launches"]), "ms": d["gpu__time_duration.sum"],
                       "dram_read": d["dram__bytes_read.sum"],
                       "dram_write": d["dram__bytes_write.sum"],
                       "dram_gbs": (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) /
                                   max(1e-9, d["gpu__time_duration.sum"]) / 1e6}
                   for k, d in sorted(per.items(), key=lambda x: -x[1]["gpu__time_duration.sum"])}}
print(json.dumps(out, indent=1))
