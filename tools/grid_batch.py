"""Time the two parts of one C2 grid batch (34 cells x 1000 C1 trees): the multi-forest
fit (aiwc_fit_cells) and the 20 prefix OOB statistics per cell (aiwc_oob_prefix_cells)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1811_00156_b200 as pkg  # noqa: E402
from paper_1811_00156_b200 import OobStatsC, _check, _p, lib, u32, vp  # noqa: E402

t = pkg.Table()
prep = pkg.PreparedDataset.from_table(t)
seed = pkg.derive_seed(1, "forest")
cps = np.arange(50, 1001, 50, dtype=np.uint32)
for first_m in (1, 18, 1):
    cells = [(m, mns) for m in range(first_m, first_m + 17) for mns in (1, 25)]
    mt = np.ascontiguousarray([c[0] for c in cells], np.uint32)
    mn = np.ascontiguousarray([c[1] for c in cells], np.uint32)
    s = time.perf_counter()
    h = vp()
    _check(lib().aiwc_fit_cells(prep._h, len(cells), _p(mt, u32), _p(mn, u32), 1000, seed, C.byref(h)))
    t1 = time.perf_counter()
    st = (OobStatsC * (len(cells) * len(cps)))()
    _check(lib().aiwc_oob_prefix_cells(prep._h, h, _p(cps, u32), len(cps), st))
    t2 = time.perf_counter()
    lib().aiwc_forest_free(h)
    t3 = time.perf_counter()
    print(f"cells m {first_m}..{first_m+16} x mns (1, 25): fit_cells {1e3*(t1-s):.1f} ms, "
          f"prefix {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms", flush=True)
