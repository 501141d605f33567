"""C2 grid_oob wall time per repetition on the C1 table (outlier probe; AIWC_PROFILE_PHASES=1 adds phases)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_1811_00156_b200 as pkg
t = pkg.Table(); prep = pkg.PreparedDataset.from_table(t)
seed = pkg.derive_seed(1, "forest")
cells = [(m, 1 + (7 * m) % 50) for m in range(1, 35)]
counts = list(range(50, 1001, 50))
for r in range(12):
    s = time.perf_counter()
    pkg.grid_oob(prep, cells, counts, seed)
    print(f"run {r}: {1e3*(time.perf_counter()-s):.1f} ms", file=sys.stderr, flush=True)
