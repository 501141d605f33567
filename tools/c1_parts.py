"""C1 config parts: 500-tree fit (OOB included) and predict_response of the 2220 rows."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_00156_b200 as pkg  # noqa: E402

t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
rows = t.predictor_rows()
p = pkg.ForestParams(500, 6, 5, pkg.derive_seed(1, "forest"))
for i in range(6):
    s0 = time.perf_counter()
    f = pkg.fit(prep, p)
    _ = f.oob
    s1 = time.perf_counter()
    _ = f.predict_response(rows)
    s2 = time.perf_counter()
    pr = f.profile()
    print(f"fit {1e3*(s1-s0):.2f} ms (grow {pr['grow_ms']:.2f}, device {pr['fit_ms']:.2f}, "
          f"launches {pr['grow_launches']}) predict {1e3*(s2-s1):.2f} ms", flush=True)
