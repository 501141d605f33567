"""Per-cell wall time of C2 grid cells, with the fit's host phases for the slow ones."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
seed = pkg.derive_seed(1, "forest")
cells = [(m, 1 + (7 * m) % 50) for m in range(1, 35)]
counts = list(range(50, 1001, 50))
for rep in range(int(os.environ.get("REPS", "2"))):
    for m, mns in cells:
        s = time.perf_counter()
        f = pkg.fit(prep, pkg.ForestParams(1000, m, mns, seed), compute_oob_stats=False)
        t1 = time.perf_counter()
        pkg.oob_prefix(f, prep, counts)
        t2 = time.perf_counter()
        del f
        t3 = time.perf_counter()
        tot = 1e3 * (t3 - s)
        if tot > 40:
            print(f"cell m={m} mns={mns}: {tot:.1f} ms = fit {1e3 * (t1 - s):.1f} + prefix "
                  f"{1e3 * (t2 - t1):.1f} + free {1e3 * (t3 - t2):.1f}", flush=True)
