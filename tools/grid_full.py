"""Full C2 grid (1,700 cells x 20 num.trees prefixes) on the C1 table, timed after the
bench's warm-up."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
seed = pkg.derive_seed(1, "forest")
counts = list(range(50, 1001, 50))
sample = [(m, 1 + (7 * m) % 50) for m in range(1, 35)]
full = [(m, mns) for m in range(1, 35) for mns in range(1, 51)]
s = time.perf_counter()
pkg.grid_oob(prep, sample + [(34, k) for k in range(1, 35)], counts, seed)
print(f"warm-up {time.perf_counter() - s:.2f} s", flush=True)
for r in range(2):
    s = time.perf_counter()
    err = pkg.grid_oob(prep, full, counts, seed)
    dt = time.perf_counter() - s
    print(f"full grid: {dt:.2f} s, {len(full) / dt:.1f} cells/s, best {err.min():.6f}", flush=True)
