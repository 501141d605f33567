"""Golden of the reference's heatmap_scan (experiments.hpp:79-123) on the C1 table, for
the drop-in batching test (tests/test_dropin.py).  TEST INFRASTRUCTURE, build container
only: runs the quarantining reference build (REFERENCE_DEFECT.md) with 8 chain threads.

    python tests/golden/make_heatmap_golden.py     # ~1-2 min on 8 cores
"""
import ctypes as C
import json
import os
import sys
import time

os.environ.setdefault("AIWC_REF_QUARANTINE", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import numpy as np  # noqa: E402
from oracle_lib import Ref, RefData  # noqa: E402

# the configuration tests/cpp/dropin_test.cpp's "heatmap" mode runs through the drop-in
CFG = dict(nt_lo=10, nt_hi=300, mt_lo=1, mt_hi=34, mns=9, max_evals=30, random_starts=8,
           sa_seed=1)


def main():
    L = Ref.lib()
    P = C.POINTER
    L.ref_heatmap.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                              C.c_int64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                              C.c_uint, P(C.c_double), C.c_uint64, P(C.c_uint64),
                              P(C.c_uint64)]
    d = RefData()
    seed = Ref.derive_seed(1, "forest")
    cap = 3 * 100000
    out = np.zeros(cap)
    nc, ne = C.c_uint64(), C.c_uint64()
    t = time.time()
    Ref.check(L.ref_heatmap(d.prepared(), CFG["nt_lo"], CFG["nt_hi"], CFG["mt_lo"],
                            CFG["mt_hi"], CFG["mns"], CFG["max_evals"], CFG["random_starts"],
                            seed, CFG["sa_seed"], 8, out.ctypes.data_as(P(C.c_double)), cap,
                            C.byref(nc), C.byref(ne)))
    cells = out[:3 * nc.value].reshape(-1, 3)
    res = {"generator": "tests/golden/make_heatmap_golden.py", "config": {**CFG, "forest_seed": seed},
           "evaluations": ne.value, "reference_s_8_threads": time.time() - t,
           "cells": [[int(a), int(b), float(c)] for a, b, c in cells]}
    with open(os.path.join(HERE, "heatmap_c1.json"), "w") as fh:
        json.dump(res, fh, indent=0)
    print(ne.value, nc.value, res["reference_s_8_threads"])


if __name__ == "__main__":
    main()
