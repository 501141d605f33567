"""One timed C4-shaped (or C1) fit through the Python mirror; for ncu launch lists.

    python tools/fit_once.py [c1|c4] [trees] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 296
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
tab = pkg.Table() if which == "c1" else pkg.Table(6757, 37)
m = 6 if which == "c1" else 8
prep = pkg.PreparedDataset.from_table(tab)
seed = pkg.derive_seed(1, "forest")
for _ in range(reps):
    s = time.perf_counter()
    f = pkg.fit(prep, pkg.ForestParams(T, m, 5, seed))
    dt = time.perf_counter() - s
    pr = f.profile()
    print(f"{which} T={T}: wall {dt*1e3:.1f} ms grow {pr['grow_ms']:.1f} ms "
          f"{T/dt:.1f} trees/s nodes/tree {f.total_nodes/T:.1f} oob {f.oob.error_pct:.9f} "
          f"split_rows {pr['split_rows']}",
          flush=True)
