"""C3 evaluate timing (505/30/9 on the C1 table), a few runs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table()
seed = pkg.derive_seed(1, "forest")
prm = pkg.ForestParams(505, 30, 9, 0)
for i in range(5):
    s = time.perf_counter()
    pred = pkg.evaluate(t, prm, seed)
    dt = time.perf_counter() - s
    err = 100.0 * np.abs(pred - t.seconds) / t.seconds
    print(f"evaluate 505/30/9: {dt*1e3:.1f} ms, {t.kernels/dt:.1f} folds/s, MAPE {err.mean():.4f} %",
          flush=True)
