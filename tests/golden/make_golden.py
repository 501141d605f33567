"""Regenerate the committed golden fixtures from the REFERENCE implementation.

Runs in the build container only (needs oracle/_ref/libaiwc_ref.so, built from
/root/reference by `make -C oracle`).  Every number here comes from the unmodified
reference headers (forest.hpp / synth.hpp / experiments.hpp) through the C-ABI shim
oracle/ref_harness.cpp.

    python tests/golden/make_golden.py            # small + C1/C3 fixtures (~1 min)
    python tests/golden/make_golden.py --c4       # + the 1M-row C4 8-tree fixture (~3 min)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Ref, RefData, RefForest, ref_evaluate  # noqa: E402


def soa_digest(s) -> str:
    h = hashlib.sha256()
    for a in (s.offsets, s.feature, s.threshold, s.left, s.right, s.value):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def inbag_digest(inbag: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(inbag, np.uint32).tobytes()).hexdigest()


def verify_tree_semantics(s, col, y, n):
    """Guard against the reference's use-after-free (oracle/REFERENCE_DEFECT.md): in a
    correctly numbered tree every node is reached by >= 1 in-bag row and every leaf holds
    the weighted mean of the in-bag responses that reach it."""
    col = np.asarray(col).reshape(-1, n)
    for t in range(s.num_trees):
        fe, th, le, ri, va = s.tree(t)
        mult = np.bincount(s.inbag[t], minlength=n).astype(np.float64)
        rows = np.nonzero(mult)[0]
        node = np.zeros(len(rows), np.int64)
        hit = np.zeros(len(fe), bool)
        while True:
            hit[np.unique(node)] = True
            sp = fe[node] >= 0
            if not sp.any():
                break
            nd, rw = node[sp], rows[sp]
            x = col[fe[nd], rw]
            node[sp] = np.where(x <= th[nd], le[nd], ri[nd])
        if not hit.all():
            raise AssertionError(f"tree {t}: unreachable nodes -> corrupted numbering")
        w = np.bincount(node, weights=mult[rows], minlength=len(fe))
        sm = np.bincount(node, weights=mult[rows] * y[rows], minlength=len(fe))
        leaf = fe < 0
        assert np.allclose(va[leaf], sm[leaf] / w[leaf], rtol=1e-9, atol=1e-12), f"tree {t}"


def checked_fit(d, T, m, mns, seed, oracle=True):
    """Reference fit, verified against the oracle (C1 sizes) or the semantic check."""
    from oracle_lib import Oracle, forests_equal
    for attempt in range(5):
        f = RefForest.fit(d, T, m, mns, seed)
        s = f.soa(d.n)
        try:
            if oracle:
                o = Oracle.fit(d.col, d.y, d.n, d.p, T, m, mns, seed)
                err = forests_equal(s, o)
                if err:
                    raise AssertionError(err)
            else:
                verify_tree_semantics(s, d.col, d.y, d.n)
            return f, s
        except AssertionError as e:
            print(f"reference fit ({T},{m},{mns}) attempt {attempt} corrupted: {e}")
    raise RuntimeError("reference kept producing corrupted forests")


def oracle_evaluate_agrees(d, T, m, mns, seed, pred_seconds) -> bool:
    """Re-run every hold-one-kernel-out fold with the oracle (experiments.hpp:393-404)."""
    from oracle_lib import Oracle
    col = d.col.reshape(d.p, d.n)
    rows = d.rows_rowmajor()
    for k in range(int(d.kernel.max()) + 1):
        tr = np.nonzero(d.kernel != k)[0]
        te = np.nonzero(d.kernel == k)[0]
        o = Oracle.fit(np.ascontiguousarray(col[:, tr]), d.y[tr], len(tr), d.p, T, m, mns,
                       Oracle.derive_seed(seed, "holdout", k))
        r = Oracle.predict(rows[te], o)
        if not np.allclose(np.power(10.0, r), pred_seconds[te], rtol=1e-13, atol=0):
            return False
    return True


def save_forest(name, s, oob, extra=None):
    np.savez_compressed(os.path.join(HERE, name + ".npz"), offsets=s.offsets, feature=s.feature,
                        threshold=s.threshold, left=s.left, right=s.right, value=s.value,
                        inbag_sha=np.frombuffer(bytes.fromhex(inbag_digest(s.inbag)), np.uint8),
                        oob=oob, **(extra or {}))


def edge_tables():
    """Small raw tables exercising the reference's edge cases."""
    rng = np.random.default_rng(7)
    out = {}
    # step dataset: y = 1 if f3 > 0.5 else 0, 100 noiseless rows
    n, p = 100, 5
    col = rng.random((p, n))
    y = (col[3] > 0.5).astype(np.float64)
    out["step"] = (col, y, dict(T=50, mtry=5, mns=1))
    # ties everywhere: few distinct values, duplicated rows, signed zeros
    n, p = 300, 7
    col = rng.integers(-2, 3, size=(p, n)).astype(np.float64)
    col[2, ::7] = -0.0
    col[2, 3::7] = 0.0
    y = rng.integers(0, 4, size=n).astype(np.float64) * 0.25 - 0.5
    out["ties"] = (col, y, dict(T=40, mtry=3, mns=2))
    # one constant column + one column constant on most rows
    n, p = 257, 4
    col = rng.normal(size=(p, n))
    col[1] = 3.0
    col[2, :250] = 1.0
    y = rng.normal(size=n)
    out["constcol"] = (col, y, dict(T=30, mtry=1, mns=1))
    # min_node_size >= n: every tree is a single leaf
    n, p = 500, 3
    col = rng.normal(size=(p, n))
    y = rng.normal(size=n)
    out["singleleaf"] = (col, y, dict(T=25, mtry=2, mns=500))
    # tiny: two rows
    col = np.array([[0.0, 1.0], [5.0, 5.0]])
    y = np.array([0.0, 1.0])
    out["tworows"] = (col, y, dict(T=8, mtry=2, mns=1))
    # mtry == p, wide table, heavy-tailed values
    n, p = 400, 40
    col = rng.standard_cauchy(size=(p, n))
    y = rng.normal(size=n) + col[0] * 1e-3
    out["wide"] = (col, y, dict(T=20, mtry=40, mns=3))
    return out


def main():
    c4 = "--c4" in sys.argv
    meta = {"generator": "tests/golden/make_golden.py", "reference": "oracle/_ref/libaiwc_ref.so"}
    seed = Ref.derive_seed(1, "forest")
    meta["forest_seed"] = seed
    d = RefData()  # C1: 37 kernels x 15 devices x 4 sizes
    meta["c1"] = {"n": d.n, "p": d.p, "fingerprint": d.fingerprint,
                  "data_sha": hashlib.sha256(d.col.tobytes() + d.y.tobytes()).hexdigest(),
                  "seconds_sha": hashlib.sha256(d.seconds.tobytes()).hexdigest(),
                  "kernel_sha": hashlib.sha256(d.kernel.tobytes()).hexdigest()}

    # C1 500/6/5: the survey golden (model JSON FNV without the trailing newline)
    f, s = checked_fit(d, 500, 6, 5, seed)
    fnv, size = f.json_fnv()
    meta["c1_500_6_5"] = {"oob": f.oob().tolist(), "json_fnv_with_newline": fnv,
                          "json_size_with_newline": size, "soa_sha": soa_digest(s),
                          "inbag_sha": inbag_digest(s.inbag),
                          "node_counts": np.diff(s.offsets).astype(int).tolist()}
    # first 20 trees in full (tree-prefix property, forest.hpp:477-479)
    k = int(s.offsets[20])
    from oracle_lib import ForestSoA
    s20 = ForestSoA(s.offsets[:21].copy(), s.feature[:k], s.threshold[:k], s.left[:k],
                    s.right[:k], s.value[:k], inbag=s.inbag[:20])
    f20, _ = checked_fit(d, 20, 6, 5, seed)
    o20 = f20.oob()
    save_forest("c1_t20_m6_n5", s20, o20)
    # predictions of the 500-tree forest on every C1 row
    pred = f.predict(d.rows_rowmajor())
    np.save(os.path.join(HERE, "c1_500_predict.npy"), pred)

    # paper params 505/30/9
    f2, s2 = checked_fit(d, 505, 30, 9, seed)
    meta["c1_505_30_9"] = {"oob": f2.oob().tolist(), "soa_sha": soa_digest(s2),
                           "inbag_sha": inbag_digest(s2.inbag)}

    # a few grid cells (C2 objective = OOB error_pct)
    cells = []
    for (T, m, mns) in [(100, 1, 1), (50, 34, 50), (150, 17, 25), (60, 42, 3), (80, 6, 9)]:
        fc, sc = checked_fit(d, T, m, mns, seed)
        cells.append({"T": T, "mtry": m, "mns": mns, "oob": fc.oob().tolist(),
                      "soa_sha": soa_digest(sc), "inbag_sha": inbag_digest(sc.inbag)})
    meta["c2_cells"] = cells

    # C3: hold-one-kernel-out evaluate at 505/30/9 and a cheaper 50/6/5
    for (T, m, mns) in [(505, 30, 9), (50, 6, 5)]:
        for attempt in range(5):
            pt, pairs, correct = ref_evaluate(d, T, m, mns, seed)
            if oracle_evaluate_agrees(d, T, m, mns, seed, pt):
                break
            print(f"reference evaluate ({T},{m},{mns}) attempt {attempt} corrupted")
        else:
            raise RuntimeError("reference evaluate kept producing corrupted folds")
        err = 100.0 * np.abs(pt - d.seconds) / d.seconds
        per_k = [float(err[d.kernel == k].mean()) for k in range(int(d.kernel.max()) + 1)]
        meta[f"c3_{T}_{m}_{mns}"] = {"pairs": pairs, "pairs_correct": correct,
                                     "mape": float(err.mean()), "mape_per_kernel": per_k,
                                     "pred_sha": hashlib.sha256(pt.tobytes()).hexdigest()}
        np.save(os.path.join(HERE, f"c3_{T}_{m}_{mns}_pred.npy"), pt)

    # raw edge-case tables
    edges = {}
    for name, (col, y, prm) in edge_tables().items():
        n, p = col.shape[1], col.shape[0]
        from oracle_lib import Oracle, forests_equal
        for attempt in range(5):
            fe = RefForest.fit_raw(col.reshape(-1), y, n, p, prm["T"], prm["mtry"], prm["mns"],
                                   seed)
            se = fe.soa(n)
            if forests_equal(se, Oracle.fit(col, y, n, p, prm["T"], prm["mtry"], prm["mns"],
                                            seed)) is None:
                break
        else:
            raise RuntimeError(f"edge table {name}: reference output corrupted")
        np.savez_compressed(os.path.join(HERE, f"edge_{name}.npz"), col=col, y=y,
                            offsets=se.offsets, feature=se.feature, threshold=se.threshold,
                            left=se.left, right=se.right, value=se.value, inbag=se.inbag,
                            oob=fe.oob())
        edges[name] = {**prm, "n": n, "p": p, "oob": fe.oob().tolist()}
    meta["edges"] = edges

    if c4:
        dd = RefData(6757, 37)
        meta["c4"] = {"n": dd.n, "p": dd.p, "fingerprint": dd.fingerprint,
                      "data_sha": hashlib.sha256(dd.col.tobytes() + dd.y.tobytes()).hexdigest()}
        f4, s4 = checked_fit(dd, 8, 8, 5, seed, oracle=False)
        meta["c4_8_8_5"] = {"oob": f4.oob().tolist(), "soa_sha": soa_digest(s4),
                            "inbag_sha": inbag_digest(s4.inbag),
                            "node_counts": np.diff(s4.offsets).astype(int).tolist(),
                            "root": [int(s4.feature[0]), float(s4.threshold[0])]}
    else:
        old = os.path.join(HERE, "golden.json")
        if os.path.exists(old):
            prev = json.load(open(old))
            for k in ("c4", "c4_8_8_5"):
                if k in prev:
                    meta[k] = prev[k]
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
