"""TEST INFRASTRUCTURE: ctypes bindings to the CPU checkers.

* ``Ref``    -> oracle/_ref/libaiwc_ref.so  (the unmodified reference headers behind
                a C-ABI shim, oracle/ref_harness.cpp; built here by oracle/Makefile and
                shipped prebuilt to the GPU box)
* ``Oracle`` -> oracle/build/liboracle.so   (the plain-C restatement, oracle/forest_oracle.c)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libaiwc_ref_q.so" if os.environ.get("AIWC_REF_QUARANTINE") else "libaiwc_ref.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "build", "liboracle.so")

u64, u32, i32, f64, vp = C.c_uint64, C.c_uint32, C.c_int32, C.c_double, C.c_void_p
P = C.POINTER


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(P(ct))


@dataclass
class ForestSoA:
    """Concatenated tree node arrays (BFS order per tree) + per-tree offsets."""

    offsets: np.ndarray  # uint64, T+1
    feature: np.ndarray  # int32
    threshold: np.ndarray  # float64
    left: np.ndarray  # int32
    right: np.ndarray  # int32
    value: np.ndarray  # float64
    inbag: np.ndarray | None = None  # uint32 T x n

    @property
    def num_trees(self) -> int:
        return len(self.offsets) - 1

    def tree(self, t: int):
        a, b = int(self.offsets[t]), int(self.offsets[t + 1])
        return (self.feature[a:b], self.threshold[a:b], self.left[a:b],
                self.right[a:b], self.value[a:b])


class Ref:
    """The reference implementation (compiled from /root/reference headers)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(REF_SO)
            L.ref_last_error.restype = C.c_char_p
            L.ref_mix64.restype = u64
            L.ref_mix64.argtypes = [u64]
            L.ref_derive_seed.restype = u64
            L.ref_derive_seed.argtypes = [u64, C.c_char_p, u64]
            L.ref_rng_bounded.argtypes = [u64, u64, u64, P(u64)]
            L.ref_synth.argtypes = [u64, u64, f64, u64, P(vp)]
            L.ref_data_free.argtypes = [vp]
            L.ref_data_rows.restype = u64
            L.ref_data_rows.argtypes = [vp]
            L.ref_data_cols.restype = u64
            L.ref_data_cols.argtypes = [vp]
            L.ref_data_export.argtypes = [vp, P(f64), P(f64), P(f64), P(u32)]
            L.ref_data_fingerprint.restype = u64
            L.ref_data_fingerprint.argtypes = [vp]
            L.ref_data_names.restype = u64
            L.ref_data_names.argtypes = [vp, C.c_char_p, u64]
            L.ref_prepare.restype = vp
            L.ref_prepare.argtypes = [vp]
            L.ref_prepared_free.argtypes = [vp]
            L.ref_fit_prepared.argtypes = [vp, u32, u32, u32, u64, C.c_uint, P(vp)]
            L.ref_grow_range.argtypes = [vp, u32, u32, u32, u64, u32, u32, C.c_uint, P(u64)]
            L.ref_fit_raw.argtypes = [P(f64), P(f64), u64, u32, u32, u32, u32, u64,
                                      C.c_uint, P(vp)]
            L.ref_forest_free.argtypes = [vp]
            L.ref_forest_trees.restype = u32
            L.ref_forest_trees.argtypes = [vp]
            L.ref_forest_nodes.restype = u64
            L.ref_forest_nodes.argtypes = [vp, u32]
            L.ref_forest_tree.argtypes = [vp, u32, P(i32), P(f64), P(i32), P(i32), P(f64)]
            L.ref_forest_inbag.argtypes = [vp, u32, P(u32)]
            L.ref_forest_oob.argtypes = [vp, P(f64)]
            L.ref_forest_json_fnv.restype = u64
            L.ref_forest_json_fnv.argtypes = [vp, P(u64)]
            L.ref_predict.argtypes = [vp, P(f64), u64, u32, C.c_uint, P(f64)]
            L.ref_evaluate.argtypes = [vp, u32, u32, u32, u64, C.c_uint, P(f64), P(u64),
                                       P(u64)]
            cls._lib = L
        return cls._lib

    @classmethod
    def check(cls, rc: int):
        if rc:
            raise RuntimeError(f"reference error {rc}: {cls.lib().ref_last_error().decode()}")

    # --- rng ---
    @classmethod
    def derive_seed(cls, seed: int, tag: str, index: int = 0) -> int:
        return cls.lib().ref_derive_seed(seed, tag.encode(), index)

    @classmethod
    def bounded_draws(cls, key: int, n: int, count: int) -> np.ndarray:
        out = np.zeros(count, np.uint64)
        cls.lib().ref_rng_bounded(key, n, count, _ptr(out, u64))
        return out


class RefData:
    """A synthesized + joined reference Dataset (synth.hpp:126, dataset.hpp:280)."""

    def __init__(self, kernels=37, devices=15, noise=0.02, seed=1):
        L = Ref.lib()
        h = vp()
        Ref.check(L.ref_synth(kernels, devices, noise, seed, C.byref(h)))
        self.h = h
        self.n = int(L.ref_data_rows(h))
        self.p = int(L.ref_data_cols(h))
        self.col = np.zeros(self.n * self.p, np.float64)
        self.y = np.zeros(self.n, np.float64)
        self.seconds = np.zeros(self.n, np.float64)
        self.kernel = np.zeros(self.n, np.uint32)
        L.ref_data_export(h, _ptr(self.col, f64), _ptr(self.y, f64),
                          _ptr(self.seconds, f64), _ptr(self.kernel, u32))
        self.fingerprint = int(L.ref_data_fingerprint(h))
        size = L.ref_data_names(h, None, 0)
        buf = C.create_string_buffer(size)
        L.ref_data_names(h, buf, size)
        self.names = buf.raw.decode().rstrip("\n").split("\n")
        self._prep = None

    def prepared(self):
        if self._prep is None:
            self._prep = Ref.lib().ref_prepare(self.h)
        return self._prep

    def rows_rowmajor(self) -> np.ndarray:
        return np.ascontiguousarray(self.col.reshape(self.p, self.n).T)

    def __del__(self):
        try:
            if self._prep is not None:
                Ref.lib().ref_prepared_free(self._prep)
            Ref.lib().ref_data_free(self.h)
        except Exception:
            pass


class RefForest:
    def __init__(self, h):
        self.h = h

    @classmethod
    def fit(cls, data: RefData, T, mtry, mns, seed, jobs=1) -> "RefForest":
        h = vp()
        Ref.check(Ref.lib().ref_fit_prepared(data.prepared(), T, mtry, mns, seed, jobs,
                                             C.byref(h)))
        return cls(h)

    @classmethod
    def fit_raw(cls, col, y, n, p, T, mtry, mns, seed, jobs=1) -> "RefForest":
        col = np.ascontiguousarray(col, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        h = vp()
        Ref.check(Ref.lib().ref_fit_raw(_ptr(col, f64), _ptr(y, f64), n, p, T, mtry, mns,
                                        seed, jobs, C.byref(h)))
        return cls(h)

    def soa(self, n: int | None = None, with_inbag=True) -> ForestSoA:
        L = Ref.lib()
        T = L.ref_forest_trees(self.h)
        counts = np.array([L.ref_forest_nodes(self.h, t) for t in range(T)], np.uint64)
        off = np.zeros(T + 1, np.uint64)
        off[1:] = np.cumsum(counts)
        N = int(off[-1])
        s = ForestSoA(off, np.zeros(N, np.int32), np.zeros(N), np.zeros(N, np.int32),
                      np.zeros(N, np.int32), np.zeros(N))
        for t in range(T):
            a = int(off[t])
            L.ref_forest_tree(self.h, t,
                              s.feature[a:].ctypes.data_as(P(i32)),
                              s.threshold[a:].ctypes.data_as(P(f64)),
                              s.left[a:].ctypes.data_as(P(i32)),
                              s.right[a:].ctypes.data_as(P(i32)),
                              s.value[a:].ctypes.data_as(P(f64)))
        if with_inbag and n is not None:
            s.inbag = np.zeros((T, n), np.uint32)
            for t in range(T):
                L.ref_forest_inbag(self.h, t, s.inbag[t].ctypes.data_as(P(u32)))
        return s

    def oob(self) -> np.ndarray:
        out = np.zeros(6)
        Ref.lib().ref_forest_oob(self.h, _ptr(out, f64))
        return out

    def json_fnv(self):
        size = u64()
        h = Ref.lib().ref_forest_json_fnv(self.h, C.byref(size))
        return int(h), int(size.value)

    def predict(self, rows: np.ndarray, jobs=0) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.float64)
        q, p = rows.shape
        out = np.zeros(q)
        Ref.lib().ref_predict(self.h, _ptr(rows, f64), q, p, jobs, _ptr(out, f64))
        return out

    def __del__(self):
        try:
            Ref.lib().ref_forest_free(self.h)
        except Exception:
            pass


def ref_evaluate(data: RefData, T, mtry, mns, seed, jobs=1):
    pred = np.zeros(data.n)
    pairs, correct = u64(), u64()
    Ref.check(Ref.lib().ref_evaluate(data.h, T, mtry, mns, seed, jobs, _ptr(pred, f64),
                                     C.byref(pairs), C.byref(correct)))
    return pred, int(pairs.value), int(correct.value)


class Oracle:
    """The plain-C restatement (oracle/forest_oracle.c)."""

    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = C.CDLL(ORACLE_SO)
            L.oracle_mix64.restype = u64
            L.oracle_mix64.argtypes = [u64]
            L.oracle_derive_seed.restype = u64
            L.oracle_derive_seed.argtypes = [u64, C.c_char_p, u64]
            L.oracle_grow_tree.restype = C.c_int64
            L.oracle_grow_tree.argtypes = [P(f64), P(f64), u64, u32, u32, u32, u64, u64,
                                           P(i32), P(f64), P(i32), P(i32), P(f64), P(u32)]
            L.oracle_oob.restype = C.c_int
            L.oracle_oob.argtypes = [P(f64), P(f64), u64, u32, u32, P(u64), P(i32), P(f64),
                                     P(i32), P(i32), P(f64), P(u32), P(f64), P(f64), P(u32)]
            L.oracle_predict.argtypes = [P(f64), u64, u32, u32, P(u64), P(i32), P(f64),
                                         P(i32), P(i32), P(f64), P(f64)]
            cls._lib = L
        return cls._lib

    @classmethod
    def derive_seed(cls, seed: int, tag: str, index: int = 0) -> int:
        return cls.lib().oracle_derive_seed(seed, tag.encode(), index)

    @classmethod
    def fit(cls, col, y, n, p, T, mtry, mns, seed, trees=None) -> ForestSoA:
        """Grow trees (default all T; `trees` = iterable of tree indices)."""
        col = np.ascontiguousarray(col, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        L = cls.lib()
        idx = list(range(T)) if trees is None else list(trees)
        parts, inb = [], np.zeros((len(idx), n), np.uint32)
        for k, t in enumerate(idx):
            f = np.zeros(2 * n, np.int32); th = np.zeros(2 * n); le = np.zeros(2 * n, np.int32)
            ri = np.zeros(2 * n, np.int32); va = np.zeros(2 * n)
            cnt = L.oracle_grow_tree(_ptr(col, f64), _ptr(y, f64), n, p, mtry, mns, seed, t,
                                     _ptr(f, i32), _ptr(th, f64), _ptr(le, i32), _ptr(ri, i32),
                                     _ptr(va, f64), _ptr(inb[k], u32))
            if cnt < 0:
                raise MemoryError("oracle allocation failed")
            parts.append((f[:cnt], th[:cnt], le[:cnt], ri[:cnt], va[:cnt]))
        off = np.zeros(len(idx) + 1, np.uint64)
        off[1:] = np.cumsum([len(x[0]) for x in parts])
        cat = [np.concatenate([x[j] for x in parts]) for j in range(5)]
        return ForestSoA(off, *cat, inbag=inb)

    @classmethod
    def oob(cls, col, y, n, p, forest: ForestSoA):
        col = np.ascontiguousarray(col, np.float64)
        y = np.ascontiguousarray(y, np.float64)
        out = np.zeros(6)
        rs = np.zeros(n)
        rc = np.zeros(n, np.uint32)
        inbag = np.ascontiguousarray(forest.inbag, np.uint32)
        rc_ = cls.lib().oracle_oob(_ptr(col, f64), _ptr(y, f64), n, p, forest.num_trees,
                                   _ptr(forest.offsets, u64), _ptr(forest.feature, i32),
                                   _ptr(forest.threshold, f64), _ptr(forest.left, i32),
                                   _ptr(forest.right, i32), _ptr(forest.value, f64),
                                   _ptr(inbag, u32), _ptr(out, f64), _ptr(rs, f64),
                                   _ptr(rc, u32))
        if rc_ == 3:
            raise RuntimeError("no out-of-bag rows: every row was in every bag")
        return out, rs, rc

    @classmethod
    def predict(cls, rows: np.ndarray, forest: ForestSoA) -> np.ndarray:
        rows = np.ascontiguousarray(rows, np.float64)
        q, p = rows.shape
        out = np.zeros(q)
        cls.lib().oracle_predict(_ptr(rows, f64), q, p, forest.num_trees,
                                 _ptr(forest.offsets, u64), _ptr(forest.feature, i32),
                                 _ptr(forest.threshold, f64), _ptr(forest.left, i32),
                                 _ptr(forest.right, i32), _ptr(forest.value, f64),
                                 _ptr(out, f64))
        return out


def forests_equal(a: ForestSoA, b: ForestSoA, check_inbag=True) -> str | None:
    """None if bit-identical structure (feature, threshold bits, children, leaf values)."""
    if a.num_trees != b.num_trees:
        return f"tree count {a.num_trees} != {b.num_trees}"
    if not np.array_equal(a.offsets, b.offsets):
        t = int(np.nonzero(a.offsets != b.offsets)[0][0]) - 1
        return f"node counts differ first at tree {t}"
    for name in ("feature", "left", "right"):
        x, y = getattr(a, name), getattr(b, name)
        if not np.array_equal(x, y):
            k = int(np.nonzero(x != y)[0][0])
            return f"{name} differs at node {k}: {x[k]} vs {y[k]}"
    for name in ("threshold", "value"):
        x, y = getattr(a, name).view(np.uint64), getattr(b, name).view(np.uint64)
        if not np.array_equal(x, y):
            k = int(np.nonzero(x != y)[0][0])
            return f"{name} bits differ at node {k}: {getattr(a, name)[k]!r} vs {getattr(b, name)[k]!r}"
    if check_inbag and a.inbag is not None and b.inbag is not None:
        if not np.array_equal(a.inbag, b.inbag):
            return "inbag differs"
    return None
