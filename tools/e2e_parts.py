"""Wall-clock parts of the C4 end-to-end path through the C-ABI (host buffers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table(6757, 37)
seed = pkg.derive_seed(1, "forest")
for rep in range(2):
    s0 = time.perf_counter()
    prep = pkg.PreparedDataset(t.col, t.y, t.n, t.p)
    s1 = time.perf_counter()
    f = pkg.fit(prep, pkg.ForestParams(1000, 8, 5, seed))
    _ = f.oob
    s2 = time.perf_counter()
    arrs = f.export()
    s3 = time.perf_counter()
    ib = f.inbag()
    s4 = time.perf_counter()
    print(f"ctx_create {s1-s0:.2f}s fit {s2-s1:.2f}s export {s3-s2:.2f}s "
          f"({sum(a.nbytes for a in arrs)/1e9:.1f} GB) inbag {s4-s3:.2f}s ({ib.nbytes/1e9:.1f} GB)",
          flush=True)
    del f, prep, arrs, ib
