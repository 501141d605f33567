"""Device-selection ranking throughput (aiwc_rank) on the C5 forest (C1 table, 1000 trees).

    python tools/rank_once.py [feature_rows]
"""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_1811_00156_b200 as pkg  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
f = pkg.fit(prep, pkg.ForestParams(1000, 6, 5, pkg.derive_seed(1, "forest")))
rows = t.predictor_rows()
feats = np.ascontiguousarray(rows[np.random.default_rng(7).integers(0, t.n, q), :27])
ndev = t.p - 27
f.rank(feats[:1000], ndev)
for _ in range(3):
    s = time.perf_counter()
    resp, best = f.rank(feats, ndev)
    el = time.perf_counter() - s
    print(f"rank q={q} x {ndev} devices: {el * 1e3:.1f} ms, {q / el / 1e6:.2f} M queries/s, "
          f"{q * ndev / el / 1e6:.1f} M device-rows/s (host buffers)")
