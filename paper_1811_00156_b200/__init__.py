"""paper_1811_00156_b200 -- B200-native random-forest path of arXiv 1811.00156 (AIWC).

Python mirror of the reference's forest API (proj/include/aiwc/forest.hpp,
experiments.hpp) over the C-ABI of ``libaiwc_cuda.so`` (include/aiwc_cuda.h):

    ForestParams            forest.hpp:22-29
    PreparedDataset         forest.hpp:458-475   (device-resident presort)
    fit(prepared, params)   forest.hpp:480-509
    Forest.predict_response forest.hpp:77-81     (batched)
    Forest.predict_time     forest.hpp:84-86
    compute_oob / oob_error forest.hpp:393, 518
    evaluate                experiments.hpp:383-408
    derive_seed             rng.hpp:32-35

Every compute call runs the sm_100a kernels; there is no CPU fallback -- the
library raises ``AiwcError`` (status 6) when no usable GPU is present and
``ImportError`` at first use when the extension has not been built.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

__all__ = [
    "AiwcError", "ParseError", "ExecutionError", "IoError", "SchemaError", "CudaError",
    "ForestParams", "OobStats", "PreparedDataset", "Forest", "Table", "fit", "compute_oob",
    "evaluate", "derive_seed", "synthesize", "lib", "device_count", "LIB_PATH",
]

LIB_PATH = os.environ.get("AIWC_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                     "libaiwc_cuda.so")

u64, u32, i32, f64, vp = C.c_uint64, C.c_uint32, C.c_int32, C.c_double, C.c_void_p
P = C.POINTER


class AiwcError(RuntimeError):
    """Base of the error taxonomy (error.hpp:10)."""

    code = 1


class ParseError(AiwcError):
    code = 2


class ExecutionError(AiwcError):
    code = 3


class IoError(AiwcError):
    code = 4


class SchemaError(AiwcError):
    code = 5


class CudaError(AiwcError):
    code = 6


_ERRORS = {2: ParseError, 3: ExecutionError, 4: IoError, 5: SchemaError, 6: CudaError}


class OobStatsC(C.Structure):
    _fields_ = [("degenerate", C.c_int32), ("mse", f64), ("response_variance", f64),
                ("error_pct", f64), ("r_squared", f64), ("rows_evaluated", u64)]


_lib = None


def lib():
    """Load libaiwc_cuda.so (fails loudly if the extension is missing)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() "
                              "(make -C paper_1811_00156_b200/csrc)")
        L = C.CDLL(LIB_PATH)
        L.aiwc_last_error.restype = C.c_char_p
        L.aiwc_version.restype = C.c_char_p
        L.aiwc_device_count.argtypes = [P(C.c_int)]
        L.aiwc_derive_seed.restype = u64
        L.aiwc_derive_seed.argtypes = [u64, C.c_char_p, u64]
        L.aiwc_ctx_create.argtypes = [P(f64), P(f64), u64, u32, C.c_int, P(vp)]
        L.aiwc_ctx_free.argtypes = [vp]
        L.aiwc_ctx_info.argtypes = [vp, P(u64), P(u32), P(C.c_int)]
        L.aiwc_fit.argtypes = [vp, u32, u32, u32, u64, u32, u32, C.c_int, P(vp)]
        L.aiwc_forest_free.argtypes = [vp]
        L.aiwc_forest_info.argtypes = [vp, P(u32), P(u64), P(u32)]
        L.aiwc_forest_node_counts.argtypes = [vp, P(u64)]
        L.aiwc_forest_export.argtypes = [vp, P(u64), P(i32), P(f64), P(i32), P(i32), P(f64)]
        L.aiwc_forest_export_inbag.argtypes = [vp, P(u32)]
        L.aiwc_forest_host_view.argtypes = [vp] + [P(vp)] * 6
        L.aiwc_forest_oob_stats.argtypes = [vp, P(OobStatsC)]
        L.aiwc_forest_import.argtypes = [u32, P(u64), P(i32), P(f64), P(i32), P(i32), P(f64),
                                         P(u32), u64, C.c_int, P(vp)]
        L.aiwc_forest_export_device.argtypes = [vp, vp, vp, vp, vp, vp]
        L.aiwc_forest_import_device.argtypes = [u32, P(u64), vp, vp, vp, vp, vp, u64, C.c_int,
                                                P(vp)]
        L.aiwc_rank.argtypes = [vp, P(f64), u64, u32, u32, P(f64), P(u32)]
        L.aiwc_oob.argtypes = [vp, vp, P(OobStatsC), P(f64), P(u32)]
        L.aiwc_oob_accumulate.argtypes = [vp, vp, P(f64), P(u32)]
        L.aiwc_oob_accumulate_device.argtypes = [vp, vp, vp, vp]
        L.aiwc_oob_finalize.argtypes = [P(f64), u64, P(f64), P(u32), P(OobStatsC)]
        L.aiwc_predict.argtypes = [vp, P(f64), u64, u32, P(f64)]
        L.aiwc_predict_device.argtypes = [vp, vp, u64, u32, vp]
        L.aiwc_evaluate.argtypes = [P(f64), P(f64), u64, u32, P(u32), u32, u32, u32, u32, u64,
                                    C.c_int, P(f64)]
        L.aiwc_evaluate_folds.argtypes = [P(f64), P(f64), u64, u32, P(u32), u32, u32, u32,
                                          u32, u32, u32, u64, C.c_int, P(f64)]
        L.aiwc_oob_prefix.argtypes = [vp, vp, P(u32), u32, P(OobStatsC)]
        L.aiwc_fit_cells.argtypes = [vp, u32, P(u32), P(u32), u32, u64, P(vp)]
        L.aiwc_oob_prefix_cells.argtypes = [vp, vp, P(u32), u32, P(OobStatsC)]
        L.aiwc_forest_profile.argtypes = [vp, P(f64), P(f64), P(u64), P(u32)]
        L.aiwc_launch_count.restype = u64
        L.aiwc_make_queries.argtypes = [vp, u64, u32, u64, u64, C.c_int, vp]
        L.aiwc_synth.argtypes = [u64, u64, f64, u64, P(vp)]
        L.aiwc_table_free.argtypes = [vp]
        L.aiwc_table_info.argtypes = [vp, P(u64), P(u32), P(u32), P(u64)]
        L.aiwc_table_export.argtypes = [vp, P(f64), P(f64), P(f64), P(u32)]
        _lib = L
    return _lib


def _check(rc: int):
    if rc:
        msg = lib().aiwc_last_error().decode()
        raise _ERRORS.get(rc, AiwcError)(f"[{rc}] {msg}")


def _p(a, ct):
    return None if a is None else a.ctypes.data_as(P(ct))


def device_count() -> int:
    c = C.c_int(0)
    _check(lib().aiwc_device_count(C.byref(c)))
    return c.value


def release_cached(device: int = 0) -> None:
    """Return the library's recycled device memory (slot arena, idle per-fit blocks,
    pool reserve) to the driver (aiwc_release_cached)."""
    _check(lib().aiwc_release_cached(device))


def derive_seed(seed: int, tag: str, index: int = 0) -> int:
    """rng.hpp:32-35"""
    return int(lib().aiwc_derive_seed(seed, tag.encode(), index))


@dataclass(frozen=True)
class ForestParams:
    """forest.hpp:22-29"""

    num_trees: int = 500
    mtry: int = 1
    min_node_size: int = 1
    seed: int = 1


@dataclass
class OobStats:
    """forest.hpp:57-64"""

    degenerate: bool = False
    mse: float = 0.0
    response_variance: float = 0.0
    error_pct: float = 0.0
    r_squared: float = 0.0
    rows_evaluated: int = 0

    @classmethod
    def _from_c(cls, s: OobStatsC) -> "OobStats":
        return cls(bool(s.degenerate), s.mse, s.response_variance, s.error_pct, s.r_squared,
                   int(s.rows_evaluated))


class Table:
    """A synthetic AIWC table in canonical order (synth.hpp:126 + dataset.hpp:280)."""

    def __init__(self, kernels=37, devices=15, noise=0.02, seed=1):
        h = vp()
        _check(lib().aiwc_synth(kernels, devices, noise, seed, C.byref(h)))
        self._h = h
        n, p, k, fp = u64(), u32(), u32(), u64()
        _check(lib().aiwc_table_info(h, C.byref(n), C.byref(p), C.byref(k), C.byref(fp)))
        self.n, self.p, self.kernels, self.fingerprint = n.value, p.value, k.value, fp.value
        self.col = np.zeros(self.n * self.p)
        self.y = np.zeros(self.n)
        self.seconds = np.zeros(self.n)
        self.kernel_of_row = np.zeros(self.n, np.uint32)
        _check(lib().aiwc_table_export(h, _p(self.col, f64), _p(self.y, f64),
                                       _p(self.seconds, f64), _p(self.kernel_of_row, u32)))
        lib().aiwc_table_free(h)
        self._h = None

    def predictor_rows(self) -> np.ndarray:
        """row-major q x p predictor rows (Dataset::predictor_row, dataset.hpp:140-148)"""
        return np.ascontiguousarray(self.col.reshape(self.p, self.n).T)


synthesize = Table


class PreparedDataset:
    """Device-resident column store + presort (forest.hpp:458-475)."""

    def __init__(self, col: np.ndarray, y: np.ndarray, n: int, p: int, device: int = 0,
                 host_mirror: bool = False):
        self.col = np.ascontiguousarray(col, np.float64).reshape(-1)
        self.y = np.ascontiguousarray(y, np.float64)
        if self.col.size != n * p or self.y.size != n:
            raise ExecutionError("column store / response sizes disagree with (n, p)")
        h = vp()
        _check(lib().aiwc_ctx_create(_p(self.col, f64), _p(self.y, f64), n, p, device,
                                     C.byref(h)))
        self._h = h
        self.n, self.p, self.device = n, p, device
        if host_mirror:  # fits stream their in-bag draws to pinned host memory as they grow
            _check(lib().aiwc_ctx_set_host_mirror(h, 1))

    @classmethod
    def from_table(cls, t: Table, device: int = 0) -> "PreparedDataset":
        return cls(t.col, t.y, t.n, t.p, device)

    def rows(self) -> int:
        return self.n

    def predictor_count(self) -> int:
        return self.p

    def close(self):
        if getattr(self, "_h", None):
            lib().aiwc_ctx_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Forest:
    """A fitted forest (forest.hpp:66-130); device-resident, host mirrors on demand."""

    def __init__(self, h, params: ForestParams | None = None, n: int = 0):
        self._h = h
        self.params = params
        self.n = n
        t, nodes, tb = u32(), u64(), u32()
        _check(lib().aiwc_forest_info(h, C.byref(t), C.byref(nodes), C.byref(tb)))
        self.num_trees, self.total_nodes, self.tree_begin = t.value, nodes.value, tb.value

    # --- Forest::trees (SoA, BFS node order per tree) ---
    def export(self, view: bool = False):
        """(offsets, feature, threshold, left, right, value).  view=True: arrays over the
        forest's own pinned host mirror (aiwc_forest_host_view: the device arrays are
        DMA'd into it once, no copy into pageable memory); they keep the forest alive."""
        if view:
            return self._host_view()[:6]
        T, N = self.num_trees, self.total_nodes
        off = np.zeros(T + 1, np.uint64)
        f = np.zeros(N, np.int32)
        th = np.zeros(N)
        le = np.zeros(N, np.int32)
        ri = np.zeros(N, np.int32)
        va = np.zeros(N)
        _check(lib().aiwc_forest_export(self._h, _p(off, u64), _p(f, i32), _p(th, f64),
                                        _p(le, i32), _p(ri, i32), _p(va, f64)))
        return off, f, th, le, ri, va

    def offsets(self) -> np.ndarray:
        off = np.zeros(self.num_trees + 1, np.uint64)
        _check(lib().aiwc_forest_export(self._h, _p(off, u64), None, None, None, None, None))
        return off

    def export_device(self, d_feature: int, d_threshold: int, d_left: int, d_value: int,
                      d_inbag: int | None = None):
        """Device-to-device copy of the node SoA (and in-bag draws) into caller buffers on
        the forest's device (aiwc_forest_export_device)."""
        _check(lib().aiwc_forest_export_device(self._h, d_feature, d_threshold, d_left,
                                               d_value, d_inbag))

    @classmethod
    def from_device(cls, offsets, d_feature: int, d_threshold: int, d_left: int, d_value: int,
                    d_inbag: int | None = None, n: int = 0, device: int = 0) -> "Forest":
        """Forest from device SoA buffers (a forest gathered over NCCL); offsets on host."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        h = vp()
        _check(lib().aiwc_forest_import_device(len(offsets) - 1, _p(offsets, u64), d_feature,
                                               d_threshold, d_left, d_value, d_inbag, n,
                                               device, C.byref(h)))
        return cls(h, None, n)

    def _host_view(self):
        ptrs = [vp() for _ in range(6)]
        _check(lib().aiwc_forest_host_view(self._h, *[C.byref(q) for q in ptrs]))
        T, N = self.num_trees, self.total_nodes

        def arr(q, count, dt, shape=None):
            if not q.value or count == 0:
                return np.zeros(shape or (count,), dt)
            raw = (C.c_char * (count * np.dtype(dt).itemsize)).from_address(q.value)
            raw._owner = self  # the forest (and its mirror) outlive the array
            a = np.frombuffer(raw, dt)
            return a.reshape(shape) if shape else a

        fe, th, le, ri, va, ib = ptrs
        return (self.offsets(), arr(fe, N, np.int32), arr(th, N, np.float64),
                arr(le, N, np.int32), arr(ri, N, np.int32), arr(va, N, np.float64),
                arr(ib, T * self.n, np.uint32, (T, self.n)) if ib.value else None)

    # --- Forest::inbag ---
    def inbag(self, view: bool = False) -> np.ndarray:
        if view:
            ib = self._host_view()[6]
            if ib is None:
                raise ExecutionError("[3] forest holds no in-bag lists")
            return ib
        out = np.zeros((self.num_trees, self.n), np.uint32)
        _check(lib().aiwc_forest_export_inbag(self._h, _p(out, u32)))
        return out

    # --- Forest::oob ---
    @property
    def oob(self) -> OobStats:
        s = OobStatsC()
        _check(lib().aiwc_forest_oob_stats(self._h, C.byref(s)))
        return OobStats._from_c(s)

    def profile(self) -> dict:
        """grow-kernel device ms, whole-fit device ms, sum of split-node rows, launches"""
        g, f, sr, gl = f64(), f64(), u64(), u32()
        _check(lib().aiwc_forest_profile(self._h, C.byref(g), C.byref(f), C.byref(sr),
                                         C.byref(gl)))
        return {"grow_ms": g.value, "fit_ms": f.value, "split_rows": sr.value,
                "grow_launches": gl.value}

    def predict_response(self, rows: np.ndarray) -> np.ndarray:
        """forest.hpp:77-81 for each row of a q x p array (or one p-vector)."""
        rows = np.ascontiguousarray(rows, np.float64)
        single = rows.ndim == 1
        rows2 = rows.reshape(1, -1) if single else rows
        q, p = rows2.shape
        out = np.zeros(q)
        _check(lib().aiwc_predict(self._h, _p(rows2, f64), q, p, _p(out, f64)))
        return out[0] if single else out

    def predict_time(self, rows: np.ndarray):
        """forest.hpp:84-86: from_response(Log10) = 10**r (dataset.hpp:89-91)"""
        return np.power(10.0, self.predict_response(rows))

    def rank(self, features: np.ndarray, ndev: int):
        """cmd_rank (tools/main.cpp:338-349) for each row of a q x nfeat feature array:
        (responses q x ndev on make_row(features, device d), best device offset q)."""
        feats = np.ascontiguousarray(features, np.float64)
        q, nfeat = feats.shape
        resp = np.zeros((q, ndev))
        best = np.zeros(q, np.uint32)
        _check(lib().aiwc_rank(self._h, _p(feats, f64), q, nfeat, ndev, _p(resp, f64),
                               _p(best, u32)))
        return resp, best

    def predict_device(self, d_rows_ptr: int, q: int, p: int, d_out_ptr: int):
        _check(lib().aiwc_predict_device(self._h, d_rows_ptr, q, p, d_out_ptr))

    @classmethod
    def from_arrays(cls, offsets, feature, threshold, left, right, value, inbag=None, n=0,
                    device=0) -> "Forest":
        """Forest::from_json equivalent from SoA arrays."""
        offsets = np.ascontiguousarray(offsets, np.uint64)
        feature = np.ascontiguousarray(feature, np.int32)
        threshold = np.ascontiguousarray(threshold, np.float64)
        left = np.ascontiguousarray(left, np.int32)
        right = np.ascontiguousarray(right, np.int32)
        value = np.ascontiguousarray(value, np.float64)
        ib = None if inbag is None else np.ascontiguousarray(inbag, np.uint32)
        h = vp()
        _check(lib().aiwc_forest_import(len(offsets) - 1, _p(offsets, u64), _p(feature, i32),
                                        _p(threshold, f64), _p(left, i32), _p(right, i32),
                                        _p(value, f64), _p(ib, u32), n, device, C.byref(h)))
        return cls(h, None, n)

    def close(self):
        if getattr(self, "_h", None):
            lib().aiwc_forest_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fit(prepared: PreparedDataset, params: ForestParams, tree_begin: int = 0,
        tree_end: int | None = None, compute_oob_stats: bool = True) -> Forest:
    """forest.hpp:480 -- grows trees [tree_begin, tree_end) (default: all) on the GPU."""
    te = params.num_trees if tree_end is None else tree_end
    h = vp()
    _check(lib().aiwc_fit(prepared._h, params.num_trees, params.mtry, params.min_node_size,
                          params.seed, tree_begin, te, 1 if compute_oob_stats else 0,
                          C.byref(h)))
    return Forest(h, params, prepared.n)


def compute_oob(forest: Forest, prepared: PreparedDataset, return_rows=False):
    """forest.hpp:393 (needs the forest's in-bag lists)."""
    s = OobStatsC()
    rs = np.zeros(prepared.n)
    rc = np.zeros(prepared.n, np.uint32)
    _check(lib().aiwc_oob(prepared._h, forest._h, C.byref(s), _p(rs, f64), _p(rc, u32)))
    st = OobStats._from_c(s)
    return (st, rs, rc) if return_rows else st


def oob_accumulate(forest: Forest, prepared: PreparedDataset, row_sum: np.ndarray,
                   row_count: np.ndarray):
    """Continue per-row tree-ordered OOB sums with this (partial) forest, in place."""
    _check(lib().aiwc_oob_accumulate(prepared._h, forest._h, _p(row_sum, f64),
                                     _p(row_count, u32)))


def oob_accumulate_device(forest: Forest, prepared: PreparedDataset, d_row_sum: int,
                          d_row_count: int):
    """oob_accumulate on device buffers (pointers: n float64, n uint32/int32 on the forest's
    device); the caller's stream must be synchronised before the call."""
    _check(lib().aiwc_oob_accumulate_device(prepared._h, forest._h, d_row_sum, d_row_count))


def oob_finalize(y: np.ndarray, row_sum: np.ndarray, row_count: np.ndarray) -> OobStats:
    y = np.ascontiguousarray(y, np.float64)
    s = OobStatsC()
    _check(lib().aiwc_oob_finalize(_p(y, f64), len(y), _p(row_sum, f64), _p(row_count, u32),
                                   C.byref(s)))
    return OobStats._from_c(s)


def launch_count() -> int:
    """kernels launched by libaiwc_cuda.so so far in this process"""
    return int(lib().aiwc_launch_count())


def make_queries(d_rows_ptr: int, n: int, p: int, q: int, seed: int, device: int,
                 d_out_ptr: int):
    """C5 queries on the device: row i copies table row Rng(derive_seed(seed,"query",i))
    .bounded(n) (device pointers, row-major)."""
    _check(lib().aiwc_make_queries(d_rows_ptr, n, p, q, seed, device, d_out_ptr))


def evaluate(table: Table, params: ForestParams, seed: int, device: int = 0,
             folds: tuple[int, int] | None = None) -> np.ndarray:
    """experiments.hpp:383-408: predicted seconds per row, each row predicted by the
    forest fit without its kernel (fold k seeded derive_seed(seed, "holdout", k)).
    `folds` = (begin, end) restricts the work to those folds (rows of other folds stay
    0.0): the per-rank share of a multi-GPU evaluate (shard.fold_range)."""
    out = np.zeros(table.n)
    fb, fe = (0, table.kernels) if folds is None else folds
    _check(lib().aiwc_evaluate_folds(_p(table.col, f64), _p(table.y, f64), table.n, table.p,
                                     _p(table.kernel_of_row, u32), table.kernels, fb, fe,
                                     params.num_trees, params.mtry, params.min_node_size,
                                     seed, device, _p(out, f64)))
    return out


def oob_prefix(forest: Forest, prepared: PreparedDataset, tree_counts) -> list:
    """OOB statistics of the forest's first T trees for each T in `tree_counts`
    (ascending): by the tree-prefix property (forest.hpp:182, 477-479) these equal
    fit(prepared, {T, mtry, mns, seed}).oob -- the grid objective of tuner.hpp:247-253
    over the num.trees axis, from one fit."""
    cps = np.ascontiguousarray(tree_counts, np.uint32)
    outs = (OobStatsC * len(cps))()
    _check(lib().aiwc_oob_prefix(prepared._h, forest._h, _p(cps, u32), len(cps), outs))
    return [OobStats._from_c(o) for o in outs]


def grid_oob(prepared: PreparedDataset, cells, tree_counts, seed: int,
             workers: int = 1, cell_batch: int = 34) -> np.ndarray:
    """C2 grid objective (tuner.hpp:247-253 / experiments.hpp:79-108): error_pct for
    every (mtry, min_node_size) cell x num.trees value, one fit of max(tree_counts)
    trees per cell.  Returns an array [len(cells), len(tree_counts)].  Tables below
    65,536 rows grow `cell_batch` cells' forests per launch (aiwc_fit_cells); larger ones
    fit cell by cell from `workers` host threads, each with its own device copy of the
    dataset (a context serialises its fits)."""
    import threading

    cps = sorted(int(t) for t in tree_counts)
    out = np.zeros((len(cells), len(cps)))
    if prepared.n < 65536 and cell_batch > 0:  # many cells' forests per launch
        cpa = np.ascontiguousarray(cps, np.uint32)
        # largest per-tree scratch first (mtry descending, min.node.size ascending): the
        # first batch sizes the device's slot arena and every later batch reuses it
        order = sorted(range(len(cells)), key=lambda i: (-cells[i][0], cells[i][1]))
        for i0 in range(0, len(cells), cell_batch):
            idx = order[i0:i0 + cell_batch]
            cs = [cells[i] for i in idx]
            mt = np.ascontiguousarray([c[0] for c in cs], np.uint32)
            mn = np.ascontiguousarray([c[1] for c in cs], np.uint32)
            h = vp()
            _check(lib().aiwc_fit_cells(prepared._h, len(cs), _p(mt, u32), _p(mn, u32), cps[-1],
                                        seed, C.byref(h)))
            try:
                st = (OobStatsC * (len(cs) * len(cps)))()
                _check(lib().aiwc_oob_prefix_cells(prepared._h, h, _p(cpa, u32), len(cps), st))
                for j, i in enumerate(idx):
                    out[i] = [st[j * len(cps) + k].error_pct for k in range(len(cps))]
            finally:
                lib().aiwc_forest_free(h)
        return out
    workers = max(1, min(workers, len(cells)))
    preps = [prepared] + [PreparedDataset(prepared.col, prepared.y, prepared.n, prepared.p,
                                          prepared.device) for _ in range(workers - 1)]
    nxt = [0]
    lock = threading.Lock()
    errors = []

    def run(prep):
        try:
            while True:
                with lock:
                    i = nxt[0]
                    nxt[0] += 1
                if i >= len(cells):
                    return
                m, mns = cells[i]
                f = fit(prep, ForestParams(cps[-1], m, mns, seed), compute_oob_stats=False)
                out[i] = [s.error_pct for s in oob_prefix(f, prep, cps)]
                del f
        except Exception as e:  # surfaced below
            errors.append(e)

    th = [threading.Thread(target=run, args=(pp,)) for pp in preps]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for pp in preps[1:]:
        pp.close()
    if errors:
        raise errors[0]
    return out
