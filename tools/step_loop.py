"""Bench-like C4 step loop (fit + OOB, forest freed each step) with per-step wall, grow
and device-fit times; run with AIWC_PROFILE_PHASES=1 for the host-side phase marks."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
t = pkg.Table(6757, 37)
prep = pkg.PreparedDataset.from_table(t)
params = pkg.ForestParams(1000, 8, 5, pkg.derive_seed(1, "forest"))
for i in range(steps):
    s = time.perf_counter()
    f = pkg.fit(prep, params)
    _ = f.oob
    w = time.perf_counter() - s
    pr = f.profile()
    del f
    print(f"step {i}: wall {w*1e3:.1f} ms grow {pr['grow_ms']:.1f} fit_dev {pr['fit_ms']:.1f} "
          f"outside_grow {w*1e3 - pr['grow_ms']:.1f}", file=sys.stderr, flush=True)
