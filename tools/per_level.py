"""Per-level kernel times of a single-lane wide fit from an ncu launch list.

    AIWC_WIDE_LANES=1 ncu --metrics gpu__time_duration.sum --csv --log-file x.csv \
        python tools/fit_once.py c4 148
    python tools/per_level.py x.csv
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
lv = -1
per = collections.defaultdict(lambda: collections.defaultdict(float))
names = []
for r in rows[start + 1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
    if k == "w_front":
        lv += 1
    if k not in names:
        names.append(k)
    per[lv][k] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-3)
keys = [k for k in ["w_chains_warp", "w_chains_grp", "w_chains_lane", "w_route", "w_lwarp",
                    "w_pay", "w_decide", "w_front"] if k in names]
print("lvl " + " ".join(f"{k[2:]:>11s}" for k in keys) + "   total(us)")
tot = collections.defaultdict(float)
for l in sorted(per):
    print(f"{l:3d} " + " ".join(f"{per[l][k]:11.0f}" for k in keys) +
          f" {sum(per[l].values()):11.0f}")
    for k in keys:
        tot[k] += per[l][k]
print("sum " + " ".join(f"{tot[k]:11.0f}" for k in keys))
