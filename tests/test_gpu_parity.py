"""GPU parity: the sm_100a forest path (through the C-ABI) against the reference goldens
(tests/golden, made by the unmodified reference) and the oracle.  Tree structure,
thresholds, leaf values and in-bag draws must be bit-identical; OOB statistics and
predictions too (the GPU sums in the reference's order, no FMA)."""
import hashlib
import os

import numpy as np
import pytest

import paper_1811_00156_b200 as pkg
from oracle_lib import ForestSoA, Oracle, forests_equal

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def soa_of(forest: pkg.Forest, with_inbag=True) -> ForestSoA:
    off, f, th, le, ri, va = forest.export()
    return ForestSoA(off, f, th, le, ri, va, inbag=forest.inbag() if with_inbag else None)


def soa_sha(s: ForestSoA) -> str:
    h = hashlib.sha256()
    for a in (s.offsets, s.feature, s.threshold, s.left, s.right, s.value):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def oob_list(st: pkg.OobStats):
    return [float(st.degenerate), st.mse, st.response_variance, st.error_pct, st.r_squared,
            float(st.rows_evaluated)]


@pytest.fixture(scope="module")
def c1():
    t = pkg.Table()
    return t, pkg.PreparedDataset.from_table(t)


@pytest.fixture(scope="module")
def seed(golden):
    return golden["forest_seed"]


def test_c1_first20_bit_exact(c1, seed):
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(20, 6, 5, seed))
    z = np.load(os.path.join(GOLD, "c1_t20_m6_n5.npz"))
    g = ForestSoA(z["offsets"], z["feature"], z["threshold"], z["left"], z["right"], z["value"])
    s = soa_of(f)
    assert forests_equal(g, s, check_inbag=False) is None
    assert hashlib.sha256(s.inbag.tobytes()).digest() == z["inbag_sha"].tobytes()
    assert oob_list(f.oob) == list(z["oob"])


def test_c1_500_forest_matches_reference(c1, seed, golden):
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(500, 6, 5, seed))
    s = soa_of(f)
    g = golden["c1_500_6_5"]
    assert np.diff(s.offsets).tolist() == g["node_counts"]
    assert soa_sha(s) == g["soa_sha"]
    assert hashlib.sha256(s.inbag.tobytes()).hexdigest() == g["inbag_sha"]
    assert oob_list(f.oob) == g["oob"]
    # batched predict_response over every C1 row, summed in tree order
    pred = f.predict_response(t.predictor_rows())
    ref = np.load(os.path.join(GOLD, "c1_500_predict.npy"))
    assert np.array_equal(pred.view(np.uint64), ref.view(np.uint64))


def test_c1_paper_params(c1, seed, golden):
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(505, 30, 9, seed))
    g = golden["c1_505_30_9"]
    s = soa_of(f)
    assert soa_sha(s) == g["soa_sha"]
    assert hashlib.sha256(s.inbag.tobytes()).hexdigest() == g["inbag_sha"]
    assert oob_list(f.oob) == g["oob"]


@pytest.mark.parametrize("cell", range(5))
def test_c2_grid_cells(c1, seed, golden, cell):
    t, prep = c1
    g = golden["c2_cells"][cell]
    f = pkg.fit(prep, pkg.ForestParams(g["T"], g["mtry"], g["mns"], seed))
    s = soa_of(f)
    assert soa_sha(s) == g["soa_sha"]
    assert oob_list(f.oob) == g["oob"]


@pytest.mark.parametrize("name", ["step", "ties", "constcol", "singleleaf", "tworows", "wide"])
def test_edge_tables(name, seed, golden):
    z = np.load(os.path.join(GOLD, f"edge_{name}.npz"))
    col, y = z["col"], z["y"]
    p, n = col.shape
    prm = golden["edges"][name]
    prep = pkg.PreparedDataset(col, y, n, p)
    f = pkg.fit(prep, pkg.ForestParams(prm["T"], prm["mtry"], prm["mns"], seed))
    g = ForestSoA(z["offsets"], z["feature"], z["threshold"], z["left"], z["right"], z["value"],
                  inbag=z["inbag"])
    assert forests_equal(g, soa_of(f)) is None
    assert oob_list(f.oob) == list(z["oob"])


def test_random_tables_vs_oracle():
    rng = np.random.default_rng(99)
    for case in range(8):
        n = int(rng.integers(2, 700))
        p = int(rng.integers(1, 20))
        col = (rng.normal(size=(p, n)) if case % 2 else
               rng.integers(0, 5, size=(p, n)).astype(float))
        y = rng.normal(size=n)
        T, m, mns = int(rng.integers(1, 16)), int(rng.integers(1, p + 1)), int(rng.integers(1, 7))
        seed = int(rng.integers(0, 2**63))
        prep = pkg.PreparedDataset(col, y, n, p)
        try:
            f = pkg.fit(prep, pkg.ForestParams(T, m, mns, seed))
        except pkg.ExecutionError as e:  # "no out-of-bag rows" like compute_oob
            assert "out-of-bag" in str(e)
            f = pkg.fit(prep, pkg.ForestParams(T, m, mns, seed), compute_oob_stats=False)
        o = Oracle.fit(col, y, n, p, T, m, mns, seed)
        assert forests_equal(o, soa_of(f)) is None, (case, n, p, T, m, mns)


def test_tree_ranges_and_chained_oob(c1, seed):
    """Sharding by tree range (the multi-GPU path) reproduces the one-shot forest and,
    with chained per-row OOB accumulation, bit-identical OOB statistics."""
    t, prep = c1
    params = pkg.ForestParams(90, 6, 5, seed)
    full = pkg.fit(prep, params)
    a = pkg.fit(prep, params, 0, 40, compute_oob_stats=False)
    b = pkg.fit(prep, params, 40, 90, compute_oob_stats=False)
    sf, sa, sb = soa_of(full), soa_of(a), soa_of(b)
    cat = ForestSoA(np.concatenate([sa.offsets, sb.offsets[1:] + sa.offsets[-1]]),
                    *(np.concatenate([getattr(sa, k), getattr(sb, k)])
                      for k in ("feature", "threshold", "left", "right", "value")),
                    inbag=np.concatenate([sa.inbag, sb.inbag]))
    assert forests_equal(sf, cat) is None
    rs = np.zeros(t.n)
    rc = np.zeros(t.n, np.uint32)
    pkg.oob_accumulate(a, prep, rs, rc)
    pkg.oob_accumulate(b, prep, rs, rc)
    assert oob_list(pkg.oob_finalize(t.y, rs, rc)) == oob_list(full.oob)


def _thread_all_gather(world):
    """In-process all_gather for `world` threads on one GPU (copies only; stands in for
    NCCL's all-gather of the multi-GPU path)."""
    import threading

    slots, bar = [None] * world, threading.Barrier(world)

    def for_rank(r):
        def ag(lst, t):
            slots[r] = t.clone()
            bar.wait()
            for i in range(world):
                lst[i].copy_(slots[i])
            bar.wait()
        return ag
    return for_rank


@pytest.mark.parametrize("with_inbag", [True, False])
def test_device_forest_gather(c1, seed, with_inbag):
    """allgather_forest (device export -> all-gather -> device import) of two ragged
    tree-range shards gives the one-shot forest on every rank: same SoA, in-bag draws,
    OOB and predictions."""
    import threading

    import torch
    from paper_1811_00156_b200 import shard

    t, prep = c1
    params = pkg.ForestParams(70, 6, 5, seed)
    full = pkg.fit(prep, params)
    parts = [pkg.fit(prep, params, 0, 31, compute_oob_stats=False),
             pkg.fit(prep, params, 31, 70, compute_oob_stats=False)]
    ag = _thread_all_gather(2)
    got, errs = [None, None], []

    def run(r):
        try:
            torch.cuda.set_device(0)
            got[r] = shard.allgather_forest(parts[r], 2, 0, ag(r), with_inbag=with_inbag)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(2)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=120)
    assert not errs, errs
    rows = t.predictor_rows()
    want = soa_of(full)
    for g in got:
        assert forests_equal(want, soa_of(g, with_inbag), check_inbag=with_inbag) is None
        assert np.array_equal(g.predict_response(rows), full.predict_response(rows))
        if with_inbag:
            assert oob_list(pkg.compute_oob(g, prep)) == oob_list(full.oob)


def test_device_import_rejects_bad_layout(c1, seed):
    import torch

    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(3, 6, 5, seed))
    s = soa_of(f, False)
    le = s.left.copy()
    le[0] = 10 ** 6  # root's children outside the tree
    d = [torch.from_numpy(np.ascontiguousarray(a)).cuda()
         for a in (s.feature, s.threshold, le, s.value)]
    with pytest.raises(pkg.ParseError):
        pkg.Forest.from_device(s.offsets, *(x.data_ptr() for x in d))


def test_rank_devices_matches_make_row_predict(c1, seed):
    """aiwc_rank (cmd_rank, tools/main.cpp:338-349): responses on the virtual
    make_row(features, device) rows equal predict on the materialised rows bit for bit, and
    the first-ranked device is the reference's (min 10^r, then device name = column)."""
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(60, 6, 5, seed))
    nfeat, ndev = 27, t.p - 27
    rows = t.predictor_rows()
    rng = np.random.default_rng(5)
    feats = np.concatenate([rows[::ndev, :nfeat],
                            rows[:40, :nfeat] * rng.uniform(0.5, 1.5, size=(40, nfeat))])
    resp, best = f.rank(feats, ndev)
    q = len(feats)
    full = np.zeros((q * ndev, t.p))
    full[:, :nfeat] = np.repeat(feats, ndev, axis=0)
    full[np.arange(q * ndev), nfeat + np.tile(np.arange(ndev), q)] = 1.0
    want = f.predict_response(full).reshape(q, ndev)
    assert np.array_equal(resp.view(np.uint64), want.view(np.uint64))
    secs = np.power(10.0, want)
    ref_best = [int(np.lexsort((np.arange(ndev), secs[i]))[0]) for i in range(q)]
    assert best.tolist() == ref_best
    # exact response ties resolve to the lowest device column
    one = pkg.fit(prep, pkg.ForestParams(1, 1, 2000, seed))  # a single leaf: all tie
    _, b1 = one.rank(feats[:4], ndev)
    assert b1.tolist() == [0, 0, 0, 0]


def test_predict_rejects_narrow_rows(c1, seed):
    """Rows narrower than the forest's split columns are a SchemaError (status 5), on the
    host-row, device-row and rank paths."""
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(30, 42, 5, seed))  # mtry = p: every column in play
    rows = t.predictor_rows()
    with pytest.raises(pkg.SchemaError):
        f.predict_response(np.ascontiguousarray(rows[:8, :20]))
    with pytest.raises(pkg.SchemaError):
        f.rank(rows[:4, :27], 3)
    assert np.array_equal(f.predict_response(rows[:8]), Oracle.predict(rows[:8], soa_of(f, False)))


def test_import_predict_and_oob(c1, seed):
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(40, 6, 5, seed))
    s = soa_of(f)
    g = pkg.Forest.from_arrays(s.offsets, s.feature, s.threshold, s.left, s.right, s.value,
                               inbag=s.inbag, n=t.n)
    rows = t.predictor_rows()
    assert np.array_equal(g.predict_response(rows), f.predict_response(rows))
    assert np.array_equal(g.predict_response(rows), Oracle.predict(rows, s))
    assert oob_list(pkg.compute_oob(g, prep)) == oob_list(f.oob)
    # arbitrary (non-training) query rows go through the f64 thresholds
    q = rows[:64] * np.random.default_rng(3).uniform(0.5, 1.5, size=(64, t.p))
    assert np.array_equal(f.predict_response(q), Oracle.predict(q, s))


def test_evaluate_c3_small(c1, seed, golden):
    t, _ = c1
    pred = pkg.evaluate(t, pkg.ForestParams(50, 6, 5, 0), seed)
    ref = np.load(os.path.join(GOLD, "c3_50_6_5_pred.npy"))
    assert np.array_equal(pred.view(np.uint64), ref.view(np.uint64))


def test_evaluate_c3_paper(c1, seed, golden):
    """C3: leave-one-kernel-out at 505/30/9 -- per-kernel MAPE of the reference."""
    t, _ = c1
    pred = pkg.evaluate(t, pkg.ForestParams(505, 30, 9, 0), seed)
    ref = np.load(os.path.join(GOLD, "c3_505_30_9_pred.npy"))
    assert np.array_equal(pred.view(np.uint64), ref.view(np.uint64))
    err = 100.0 * np.abs(pred - t.seconds) / t.seconds
    g = golden["c3_505_30_9"]
    assert err.mean() == g["mape"]


def test_parameter_errors(c1):
    t, prep = c1
    with pytest.raises(pkg.ExecutionError, match="mtry"):
        pkg.fit(prep, pkg.ForestParams(5, t.p + 1, 5, 1))
    with pytest.raises(pkg.ExecutionError, match="num_trees"):
        pkg.fit(prep, pkg.ForestParams(0, 2, 5, 1))
    with pytest.raises(pkg.ExecutionError, match="min_node_size"):
        pkg.fit(prep, pkg.ForestParams(5, 2, 0, 1))


def test_degenerate_response():
    n, p = 50, 3
    col = np.random.default_rng(1).normal(size=(p, n))
    prep = pkg.PreparedDataset(col, np.full(n, 0.25), n, p)
    f = pkg.fit(prep, pkg.ForestParams(10, 2, 1, 3))
    assert f.oob.degenerate


@pytest.mark.slow
def test_c4_first8_trees(seed, golden):
    """C4 (1,000,036 x 64): first 8 trees of the 1000-tree m=8 mns=5 forest."""
    t = pkg.Table(6757, 37)
    prep = pkg.PreparedDataset.from_table(t)
    f = pkg.fit(prep, pkg.ForestParams(8, 8, 5, seed))
    g = golden["c4_8_8_5"]
    s = soa_of(f)
    assert np.diff(s.offsets).tolist() == g["node_counts"]
    assert soa_sha(s) == g["soa_sha"]
    assert hashlib.sha256(s.inbag.tobytes()).hexdigest() == g["inbag_sha"]
    assert oob_list(f.oob) == g["oob"]


@pytest.mark.parametrize("path", ["wide", "persistent"])
def test_both_growers_bit_exact(path, seed, golden, monkeypatch):
    """The batched wide grower (default for n >= 65536) and the per-tree persistent
    grower (default below) produce the same forests; force each on C1 and edge tables."""
    monkeypatch.setenv("AIWC_GROW_WIDE", "1" if path == "wide" else "0")
    t = pkg.Table()
    prep = pkg.PreparedDataset.from_table(t)
    f = pkg.fit(prep, pkg.ForestParams(60, 6, 5, seed))
    s = soa_of(f)
    o = Oracle.fit(t.col, t.y, t.n, t.p, 60, 6, 5, seed)
    assert forests_equal(o, s) is None
    for name in ("ties", "tworows", "constcol"):
        z = np.load(os.path.join(GOLD, f"edge_{name}.npz"))
        col, y = z["col"], z["y"]
        p, n = col.shape
        prm = golden["edges"][name]
        f = pkg.fit(pkg.PreparedDataset(col, y, n, p),
                    pkg.ForestParams(prm["T"], prm["mtry"], prm["mns"], seed))
        g = ForestSoA(z["offsets"], z["feature"], z["threshold"], z["left"], z["right"],
                      z["value"], inbag=z["inbag"])
        assert forests_equal(g, soa_of(f)) is None


def test_wide_grower_random_tables(seed, monkeypatch):
    """The wide grower's chain kernels (lane / lane-group / warp per chain) on random
    tables mixing continuous, tied and two-level columns, over the whole mtry range
    (group widths 32..1 and several groups per node when mtry > 32)."""
    monkeypatch.setenv("AIWC_GROW_WIDE", "1")
    rng = np.random.default_rng(1811)
    cases = [(1, 1), (2, 2), (5, 3), (9, 8), (20, 16), (40, 33), (70, 64), (34, 6)]
    for case, (p, m) in enumerate(cases):
        n = int(rng.integers(300, 2500))
        kinds = rng.integers(0, 3, size=p)
        col = np.empty((p, n))
        for c in range(p):
            if kinds[c] == 0:
                col[c] = rng.normal(size=n)
            elif kinds[c] == 1:
                col[c] = rng.integers(0, 7, size=n).astype(float)
            else:
                col[c] = rng.integers(0, 2, size=n).astype(float)
        y = rng.normal(size=n)
        T, mns = 6, int(rng.integers(1, 6))
        # big-node chains from 64 rows with 16 / 8 / 32 lanes per chain | CTA chains +
        # routes from 200 rows | lane groups only
        for big_min, coop_min, lanes in (("64", "1000000", "16"), ("64", "1000000", "8"),
                                         ("64", "1000000", "32"), ("64", "200", "16"),
                                         ("1000000", "1000000", "16")):
            # the list pass with the bitmap in global memory (the path of tables whose
            # bitmap exceeds shared memory) on the last configuration
            if big_min == "1000000":
                monkeypatch.setenv("AIWC_LW_GLOBAL", "1")
            else:
                monkeypatch.delenv("AIWC_LW_GLOBAL", raising=False)
            monkeypatch.setenv("AIWC_BIG_MIN", big_min)
            monkeypatch.setenv("AIWC_COOP_MIN", coop_min)
            monkeypatch.setenv("AIWC_BIG_LANES", lanes)
            monkeypatch.setenv("AIWC_LANE_MAX", "48" if lanes == "8" else "16")
            prep = pkg.PreparedDataset(col, y, n, p)
            f = pkg.fit(prep, pkg.ForestParams(T, m, mns, seed))
            o = Oracle.fit(col, y, n, p, T, m, mns, seed)
            assert forests_equal(o, soa_of(f)) is None, (case, n, p, m, mns, big_min, coop_min,
                                                         lanes)


def test_oob_prefix_equals_separate_fits(c1, seed, golden):
    """Tree-prefix OOB (one 500-tree fit) == the OOB of separate T-tree fits, and the
    500-tree value == the reference golden (C1 500/6/5)."""
    t, prep = c1
    counts = [1, 7, 50, 123, 500]
    f = pkg.fit(prep, pkg.ForestParams(500, 6, 5, seed), compute_oob_stats=False)
    pre = pkg.oob_prefix(f, prep, counts)
    for T, st in zip(counts[:-1], pre):
        want = pkg.fit(prep, pkg.ForestParams(T, 6, 5, seed)).oob
        assert oob_list(st) == oob_list(want), T
    assert pre[-1].error_pct == golden["c1_500_6_5"]["oob"][3]


def test_grid_oob_matches_reference_cells(c1, seed, golden):
    """C2 objective through grid_oob on the reference's golden grid cells."""
    t, prep = c1
    for g in golden["c2_cells"]:
        got = pkg.grid_oob(prep, [(g["mtry"], g["mns"])], [g["T"] // 2, g["T"]], seed)
        assert got[0, 1] == g["oob"][3], g


def test_evaluate_fold_ranges_combine(c1, seed):
    """The multi-GPU split of evaluate: fold ranges of two ranks, summed row-wise, equal
    the whole evaluate bit-for-bit (C3 at 50/6/5 against the reference golden)."""
    from paper_1811_00156_b200 import shard
    t, _ = c1
    prm = pkg.ForestParams(50, 6, 5, 0)
    parts = [pkg.evaluate(t, prm, seed, folds=shard.fold_range(r, 2, t.kernels))
             for r in range(2)]
    ref = np.load(os.path.join(GOLD, "c3_50_6_5_pred.npy"))
    assert np.array_equal((parts[0] + parts[1]).view(np.uint64), ref.view(np.uint64))


def test_wide_grower_u32_ranks(seed):
    """A column with more than 65,536 distinct values switches the rank table to u32;
    the wide grower (default for n >= 65,536) must stay bit-exact on it."""
    rng = np.random.default_rng(4242)
    n, p = 70_000, 3
    col = np.vstack([rng.normal(size=n), rng.integers(0, 9, size=n).astype(float),
                     rng.integers(0, 2, size=n).astype(float)])
    y = rng.normal(size=n)
    prep = pkg.PreparedDataset(col, y, n, p)
    f = pkg.fit(prep, pkg.ForestParams(3, 2, 5, seed))
    o = Oracle.fit(col, y, n, p, 3, 2, 5, seed)
    assert forests_equal(o, soa_of(f)) is None
    stats, _, _ = Oracle.oob(col, y, n, p, o)
    assert [f.oob.mse, f.oob.error_pct] == [stats[1], stats[3]]


def test_grid_cells_batched_equal_separate_fits(c1, seed):
    """aiwc_fit_cells (per-tree mtry / min.node.size, one launch) == one fit per cell:
    every prefix OOB statistic bit-for-bit, over cells with different tree shapes."""
    t, prep = c1
    cells = [(1, 1), (6, 5), (42, 50), (17, 3), (30, 9)]
    counts = [1, 13, 40]
    got = pkg.grid_oob(prep, cells, counts, seed, cell_batch=3)  # 120 trees: wide grower
    # the CTA-per-tree grower takes the same cells (few trees per launch)
    os.environ["AIWC_GROW_WIDE"] = "0"
    try:
        got0 = pkg.grid_oob(prep, cells, counts, seed, cell_batch=5)
    finally:
        del os.environ["AIWC_GROW_WIDE"]
    assert np.array_equal(got, got0)
    for i, (m, mns) in enumerate(cells):
        f = pkg.fit(prep, pkg.ForestParams(counts[-1], m, mns, seed), compute_oob_stats=False)
        want = [s.error_pct for s in pkg.oob_prefix(f, prep, counts)]
        assert list(got[i]) == want, (m, mns)


def test_evaluate_ragged_interleaved_folds(c1, seed):
    """Fold-batched evaluate (all folds as one multi-forest launch on one device copy of
    the table, each fold bootstrapping from its own training rows) on folds that are
    neither contiguous nor equal-sized: every held-out row equals the oracle's forest fit
    on that fold's training subset (experiments.hpp:393-402), predict_time with pow."""
    import math

    from paper_1811_00156_b200 import _check, _p, f64, lib, u32

    t, _ = c1
    K, T, m, mns = 4, 24, 6, 5
    label = ((np.arange(t.n) * 7) // 13 % K).astype(np.uint32)
    label[label == 3] = np.where(np.arange(t.n)[label == 3] % 3 == 0, 3, 1)  # uneven sizes
    out = np.zeros(t.n)
    _check(lib().aiwc_evaluate_folds(_p(t.col, f64), _p(t.y, f64), t.n, t.p, _p(label, u32), K,
                                     0, K, T, m, mns, seed, 0, _p(out, f64)))
    col = t.col.reshape(t.p, t.n)
    rows_all = t.predictor_rows()
    for k in range(K):
        tr = np.flatnonzero(label != k)
        te = np.flatnonzero(label == k)
        sub = np.ascontiguousarray(col[:, tr]).reshape(-1)
        want = Oracle.fit(sub, t.y[tr], len(tr), t.p, T, m, mns, pkg.derive_seed(seed, "holdout", k))
        resp = Oracle.predict(rows_all[te], want)
        exp = np.array([math.pow(10.0, r) for r in resp])
        assert np.array_equal(out[te].view(np.uint64), exp.view(np.uint64)), f"fold {k}"


def test_host_view_equals_export(c1, seed):
    """aiwc_forest_host_view (pinned host mirror, zero-copy numpy views) holds exactly the
    arrays the copying export returns."""
    t, prep = c1
    f = pkg.fit(prep, pkg.ForestParams(64, 6, 5, seed))
    a = f.export()
    v = f.export(view=True)
    for x, y in zip(a, v):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    assert np.array_equal(f.inbag(), f.inbag(view=True))
    ib = f.inbag(view=True)
    del f  # the views keep the forest (and its mirror) alive
    assert ib.shape == (64, t.n) and int(ib.sum()) > 0


@pytest.mark.parametrize("trees", [16, 200])
def test_fit_time_inbag_mirror(c1, seed, trees):
    """host_mirror datasets stream each batch's in-bag draws to pinned memory during the fit
    (both growers: 16 trees take the CTA-per-tree one, 200 the batched one); the host view
    equals the copying export, and the forest equals the same fit without the mirror."""
    t, prep = c1
    pm = pkg.PreparedDataset(t.col, t.y, t.n, t.p, host_mirror=True)
    params = pkg.ForestParams(trees, 6, 5, seed)
    f = pkg.fit(pm, params)
    g = pkg.fit(prep, params)
    assert np.array_equal(f.inbag(view=True), g.inbag())
    for x, y in zip(f.export(view=True), g.export()):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))


def test_release_cached_between_fits(c1, seed):
    """aiwc_release_cached returns the recycled device / pinned memory while forests and
    their host views stay valid; the next fit re-allocates and grows the same forest."""
    t, prep = c1
    params = pkg.ForestParams(100, 6, 5, seed)
    f = pkg.fit(prep, params)
    view = f.export(view=True)
    pkg.release_cached(0)
    g = pkg.fit(prep, params)
    for x, y in zip(view, g.export()):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
