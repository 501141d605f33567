"""C5 predict timing: 1000-tree C1 forest over Q device-resident queries, checked
against the oracle on a sample.

    python tools/predict_once.py [Q] [reps]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_00156_b200 as pkg  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
f = pkg.fit(prep, pkg.ForestParams(1000, 6, 5, pkg.derive_seed(1, "forest")))
rows = torch.from_numpy(t.predictor_rows()).cuda()
qbuf = torch.empty((q, t.p), dtype=torch.float64, device="cuda")
out = torch.empty(q, dtype=torch.float64, device="cuda")
pkg.make_queries(rows.data_ptr(), t.n, t.p, q, 7, 0, qbuf.data_ptr())
f.predict_device(qbuf.data_ptr(), q, t.p, out.data_ptr())
torch.cuda.synchronize()
# parity on the first 4096 queries against the oracle's walk (forest.hpp:42-50, 77-81)
from oracle_lib import ForestSoA, Oracle  # noqa: E402
off, fe, th, le, ri, va = f.export()
want = Oracle.predict(qbuf[:4096].cpu().numpy(), ForestSoA(off, fe, th, le, ri, va))
assert np.array_equal(out[:4096].cpu().numpy(), want), "predict mismatch"
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.predict_device(qbuf.data_ptr(), q, t.p, out.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"predict q={q}: {ms:.1f} ms, {q / ms * 1e3 / 1e6:.1f} M rows/s", flush=True)
