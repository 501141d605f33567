"""C5 predict end to end through aiwc_predict (host rows in, host responses out)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1811_00156_b200 as pkg  # noqa: E402

q = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
t = pkg.Table()
f = pkg.fit(pkg.PreparedDataset.from_table(t), pkg.ForestParams(1000, 6, 5, pkg.derive_seed(1, "forest")))
rows = torch.from_numpy(t.predictor_rows()).cuda()
qbuf = torch.empty((q, t.p), dtype=torch.float64, device="cuda")
pkg.make_queries(rows.data_ptr(), t.n, t.p, q, 7, 0, qbuf.data_ptr())
out = torch.empty(q, dtype=torch.float64, device="cuda")
f.predict_device(qbuf.data_ptr(), q, t.p, out.data_ptr())
host = qbuf.cpu().numpy()
for _ in range(3):
    s = time.perf_counter()
    r = f.predict_response(host)
    dt = time.perf_counter() - s
    print(f"e2e q={q}: {dt*1e3:.0f} ms, {q/dt/1e6:.1f} M rows/s, "
          f"equal to device path: {np.array_equal(r, out.cpu().numpy())}", flush=True)
