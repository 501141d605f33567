"""Fit timing + per-phase cycle shares of the grower (AIWC_PROFILE_PHASES=1).

    python tools/prof_fit.py [c1|c4] [trees] [mtry] [mns]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("AIWC_PROFILE_PHASES", "1")
import paper_1811_00156_b200 as pkg  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c1"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 500
t0 = time.perf_counter()
tab = {"c1": lambda: pkg.Table(), "c4": lambda: pkg.Table(6757, 37),
       "c4s": lambda: pkg.Table(1500, 37)}[which]()
m = int(sys.argv[3]) if len(sys.argv) > 3 else (6 if which == "c1" else 8)
mns = int(sys.argv[4]) if len(sys.argv) > 4 else 5
prep = pkg.PreparedDataset.from_table(tab)
print(f"setup {time.perf_counter() - t0:.2f}s n={tab.n} p={tab.p}", flush=True)
seed = pkg.derive_seed(1, "forest")
for rep in range(2):
    s = time.perf_counter()
    f = pkg.fit(prep, pkg.ForestParams(T, m, mns, seed))
    dt = time.perf_counter() - s
    pr = f.profile()
    print(f"{which} T={T} m={m} mns={mns}: wall {dt*1e3:.1f} ms, grow {pr['grow_ms']:.1f} ms, "
          f"fit {pr['fit_ms']:.1f} ms, {T/dt:.1f} trees/s, nodes/tree {f.total_nodes/T:.1f}, "
          f"oob {f.oob.error_pct:.6f}", flush=True)
