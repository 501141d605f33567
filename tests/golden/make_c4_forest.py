"""Pin the whole 1000-tree C4 forest (BASELINE configs[3]) from the REFERENCE.

TEST INFRASTRUCTURE, build container only (needs oracle/_ref/libaiwc_ref.so).  The
reference's multi-threaded fit is nondeterministic (oracle/REFERENCE_DEFECT.md), so
every tree is grown single-threaded by the quarantining build of the reference
(freed blocks are held back from malloc, so its dangling read sees intact data) (ref_grow_tree_oob -> TreeGrower::grow,
forest.hpp:179-376) in one of W worker PROCESSES (no allocator sharing), each over a
contiguous tree range.  Each worker also walks its trees' out-of-bag rows exactly as
compute_oob does (forest.hpp:418-433) and stores the per-row leaf values; the combine
step then sums them in tree order (the reference's sum[i] += leaf, t ascending) and
finalises the statistics as forest.hpp:396-453 does.

    python tests/golden/make_c4_forest.py run --workers 7      # ~35 min on 8 cores
    python tests/golden/make_c4_forest.py combine              # -> c4_forest_1000.json

Output `tests/golden/c4_forest_1000.json`: per-tree node count and SHA-256 of the node
arrays (feature i32 | threshold f64 | left i32 | right i32 | value f64, BFS order), the
in-bag SHA-256 of every 50th tree, and the forest's OOB statistics.
"""
from __future__ import annotations

import argparse
import ctypes as C
import hashlib
import json
import os
import subprocess
import sys
import time

import numpy as np

# the quarantining reference build (oracle/Makefile libaiwc_ref_q.so): deterministic,
# intended semantics whatever the heap state (REFERENCE_DEFECT.md)
os.environ.setdefault("AIWC_REF_QUARANTINE", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Ref, RefData  # noqa: E402

T, MTRY, MNS = 1000, 8, 5
WORK = os.environ.get("AIWC_C4_WORK", "/tmp/aiwc_c4_forest")
P = C.POINTER


def tree_digest(fe, th, le, ri, va) -> str:
    h = hashlib.sha256()
    for a, dt in ((fe, np.int32), (th, np.float64), (le, np.int32), (ri, np.int32),
                  (va, np.float64)):
        h.update(np.ascontiguousarray(a, dt).tobytes())
    return h.hexdigest()


def worker(t0: int, t1: int):
    L = Ref.lib()
    L.ref_grow_tree_oob.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32,
                                    C.c_uint64, C.c_uint32, P(C.c_double), C.c_uint64,
                                    P(C.c_uint64), P(C.c_int32), P(C.c_double),
                                    P(C.c_int32), P(C.c_int32), P(C.c_double),
                                    P(C.c_uint32)]
    d = RefData(6757, 37)
    prep = d.prepared()
    seed = Ref.derive_seed(1, "forest")
    n = d.n
    cap = 2 * n
    fe = np.zeros(cap, np.int32)
    th = np.zeros(cap)
    le = np.zeros(cap, np.int32)
    ri = np.zeros(cap, np.int32)
    va = np.zeros(cap)
    inbag = np.zeros(n, np.uint32)
    oob = np.zeros(n)
    for t in range(t0, t1):
        out = os.path.join(WORK, f"tree_{t:04d}.json")
        if os.path.exists(out):
            continue
        nodes = C.c_uint64()
        Ref.check(L.ref_grow_tree_oob(
            prep, T, MTRY, MNS, seed, t, oob.ctypes.data_as(P(C.c_double)), cap,
            C.byref(nodes), fe.ctypes.data_as(P(C.c_int32)), th.ctypes.data_as(P(C.c_double)),
            le.ctypes.data_as(P(C.c_int32)), ri.ctypes.data_as(P(C.c_int32)),
            va.ctypes.data_as(P(C.c_double)), inbag.ctypes.data_as(P(C.c_uint32))))
        k = nodes.value
        np.save(os.path.join(WORK, f"oob_{t:04d}.npy"), oob)
        rec = {"t": t, "nodes": int(k), "sha": tree_digest(fe[:k], th[:k], le[:k], ri[:k], va[:k]),
               "inbag_sha": hashlib.sha256(inbag.tobytes()).hexdigest(),
               "root": [int(fe[0]), float(th[0])]}
        with open(out + ".tmp", "w") as fh:
            json.dump(rec, fh)
        os.replace(out + ".tmp", out)
        print(f"tree {t}: {k} nodes", flush=True)


def run(workers: int):
    os.makedirs(WORK, exist_ok=True)
    bounds = [round(i * T / workers) for i in range(workers + 1)]
    procs = []
    for w in range(workers):
        log = open(os.path.join(WORK, f"worker_{w}.log"), "w")
        procs.append(subprocess.Popen([sys.executable, __file__, "worker", str(bounds[w]),
                                       str(bounds[w + 1])], stdout=log, stderr=log))
    for p in procs:
        p.wait()
    print("workers:", [p.returncode for p in procs])


def combine():
    d = RefData(6757, 37)
    n, y = d.n, d.y
    s = np.zeros(n)
    cnt = np.zeros(n, np.uint32)
    trees = []
    for t in range(T):
        rec = json.load(open(os.path.join(WORK, f"tree_{t:04d}.json")))
        trees.append(rec)
        v = np.load(os.path.join(WORK, f"oob_{t:04d}.npy"))
        m = ~np.isnan(v)
        s = s + np.where(m, v, 0.0)  # +0.0 for in-bag rows: exact (s starts at +0.0)
        cnt += m
    # forest.hpp:396-405 / 436-453 (row-order loops: sequential Python floats)
    mean = 0.0
    for v in y.tolist():
        mean += v
    mean /= n
    var = 0.0
    for v in y.tolist():
        var += (v - mean) * (v - mean)
    var /= n
    mse = 0.0
    ev = 0
    for i in np.nonzero(cnt)[0].tolist():
        pred = s[i] / float(cnt[i])
        mse += (pred - y[i]) * (pred - y[i])
        ev += 1
    mse /= ev
    out = {"generator": "tests/golden/make_c4_forest.py", "reference": "oracle/_ref/libaiwc_ref.so",
           "config": {"kernels": 6757, "devices": 37, "n": n, "p": d.p, "trees": T,
                      "mtry": MTRY, "mns": MNS, "seed": Ref.derive_seed(1, "forest")},
           "oob": {"mse": mse, "response_variance": var, "error_pct": 100.0 * mse / var,
                   "r_squared": 1.0 - mse / var, "rows_evaluated": ev},
           "oob_sum_sha": hashlib.sha256(s.tobytes()).hexdigest(),
           "oob_count_sha": hashlib.sha256(cnt.tobytes()).hexdigest(),
           "node_counts": [r["nodes"] for r in trees],
           "tree_sha": [r["sha"] for r in trees],
           "inbag_sha_every50": {str(r["t"]): r["inbag_sha"] for r in trees if r["t"] % 50 == 0}}
    with open(os.path.join(HERE, "c4_forest_1000.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(json.dumps(out["oob"]))


if __name__ == "__main__":
    if sys.argv[1] == "worker":
        worker(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    ap = argparse.ArgumentParser()
    ap.add_argument("cmd", choices=["run", "combine"])
    ap.add_argument("--workers", type=int, default=7)
    a = ap.parse_args()
    t = time.time()
    run(a.workers) if a.cmd == "run" else combine()
    print(f"{time.time() - t:.0f} s")
