"""Wall-clock parts of the C4 end-to-end path (host buffers), with fresh vs pre-faulted
output arrays, to see where the e2e time beyond the grow phase goes."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
t = pkg.Table(6757, 37)
seed = pkg.derive_seed(1, "forest")
for rep in range(3):
    s0 = time.perf_counter()
    prep = pkg.PreparedDataset(t.col, t.y, t.n, t.p)
    s1 = time.perf_counter()
    f = pkg.fit(prep, pkg.ForestParams(T, 8, 5, seed))
    _ = f.oob
    s2 = time.perf_counter()
    arrs = f.export()
    s3 = time.perf_counter()
    ib = f.inbag()
    s4 = time.perf_counter()
    N = f.total_nodes
    pre = [np.ones(N, np.int32) for _ in range(3)] + [np.ones(N) for _ in range(2)]
    ibp = np.ones((f.num_trees, f.n), np.uint32)
    off = np.zeros(f.num_trees + 1, np.uint64)
    s5 = time.perf_counter()
    L = pkg.lib()
    P = pkg._p
    pkg._check(L.aiwc_forest_export(f._h, P(off, pkg.u64), P(pre[0], pkg.i32), P(pre[3], pkg.f64),
                                    P(pre[1], pkg.i32), P(pre[2], pkg.i32), P(pre[4], pkg.f64)))
    s6 = time.perf_counter()
    pkg._check(L.aiwc_forest_export_inbag(f._h, P(ibp, pkg.u32)))
    s7 = time.perf_counter()
    pr = f.profile()
    print(f"rep {rep}: ctx_create {s1-s0:.3f}s fit {s2-s1:.3f}s (grow {pr['grow_ms']/1e3:.3f} "
          f"fit_dev {pr['fit_ms']/1e3:.3f}) export {s3-s2:.3f}s "
          f"({sum(a.nbytes for a in arrs)/1e9:.2f} GB) inbag {s4-s3:.3f}s ({ib.nbytes/1e9:.2f} GB) | "
          f"prefaulted export {s6-s5:.3f}s inbag {s7-s6:.3f}s", flush=True)
    del f, prep, arrs, ib, pre, ibp
