"""Per-kernel share of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_share.py gpurun_out/launches.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
im = h.index("Metric Name")
scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3,
         "ms": 1.0}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[start + 1:]:
    if len(r) <= iv or r[im] != "gpu__time_duration.sum":
        continue
    k = r[ik].split("(")[0].replace("void ", "").replace("aiwc_b200::", "")
    agg[k][0] += 1
    agg[k][1] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'ms':>10s} {'share':>7s}")
for k, (c, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:48]:48s} {c:8d} {ms:10.2f} {100 * ms / tot:6.2f}%")
print(f"{'total':48s} {'':8s} {tot:10.2f}")
