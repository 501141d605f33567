"""Time the parts of C2 grid cells (1000-tree C1 fit + 20 prefix OOB statistics)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
seed = pkg.derive_seed(1, "forest")
counts = list(range(50, 1001, 50))
for m, mns in ((17, 20), (17, 20), (5, 1), (30, 45), (6, 5)):
    s = time.perf_counter()
    f = pkg.fit(prep, pkg.ForestParams(1000, m, mns, seed), compute_oob_stats=False)
    t1 = time.perf_counter()
    pkg.oob_prefix(f, prep, counts)
    t2 = time.perf_counter()
    pr = f.profile()
    print(f"m={m} mns={mns}: fit {1e3 * (t1 - s):.1f} ms (grow {pr['grow_ms']:.1f}, device "
          f"{pr['fit_ms']:.1f}), prefix {1e3 * (t2 - t1):.1f} ms, "
          f"{f.total_nodes / 1000:.0f} nodes/tree", flush=True)
