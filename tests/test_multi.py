"""CPU, world_size 2 (gloo): the multi-GPU host path of paper_1811_00156_b200/shard.py.

Each rank grows its tree range of the global forest (the oracle stands in for the
per-rank GPU fit on this CPU-only box), the OOB per-row sums are chained rank 0 -> 1
over torch.distributed send/recv, and the forest parts are gathered in rank order.
The result must equal a single-process fit bit-for-bit (structure, in-bag lists, OOB
statistics) -- the property bench.py relies on for --gpus N."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle_lib import ForestSoA, Oracle, forests_equal

HERE = os.path.dirname(os.path.abspath(__file__))


def _table():
    z = np.load(os.path.join(HERE, "golden", "edge_ties.npz"))
    return z["col"], z["y"]


def _walk_rows(s: ForestSoA, t: int, col: np.ndarray) -> np.ndarray:
    fe, th, le, _, va = s.tree(t)
    n = col.shape[1]
    node = np.zeros(n, np.int64)
    while True:
        sp = fe[node] >= 0
        if not sp.any():
            return va[node]
        nd = node[sp]
        x = col[fe[nd], np.nonzero(sp)[0]]
        node[sp] = np.where(x <= th[nd], le[nd], le[nd] + 1)


def _oracle_accumulate(part: ForestSoA, col: np.ndarray):
    """Continue per-row tree-ordered OOB sums with the trees of `part` (the role of
    aiwc_oob_accumulate on a GPU rank)."""
    n = col.shape[1]

    def acc(rs, rc):
        for t in range(part.num_trees):
            bag = np.zeros(n, bool)
            bag[part.inbag[t]] = True
            leaf = _walk_rows(part, t, col)
            for i in np.nonzero(~bag)[0]:  # row order; each row's sum in tree order
                rs[i] += leaf[i]
                rc[i] += 1
    return acc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, m, mns, seed, q):
    from paper_1811_00156_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        col, y = _table()
        p, n = col.shape
        t0, t1 = shard.tree_range(rank, world, T)
        part = Oracle.fit(col, y, n, p, T, m, mns, seed, trees=range(t0, t1))
        send, recv = shard.torch_transport()
        res = shard.chained_oob(n, rank, world, _oracle_accumulate(part, col), send, recv)
        import torch

        arrays = [torch.from_numpy(np.ascontiguousarray(a)) for a in
                  (part.feature, part.threshold, part.left, part.value,
                   part.inbag.reshape(-1).view(np.int32))]
        off, g = shard.gather_forest(part.offsets, arrays, world, dist.all_gather, n)
        fe, th, le, va, ib = (t.numpy() for t in g)
        ri = np.where(le < 0, -1, le + 1).astype(np.int32)
        gathered = (off, fe, th, le, ri, va, ib.view(np.uint32).reshape(-1, n))
        if rank == world - 1:
            from paper_1811_00156_b200 import oob_finalize  # host-only C-ABI function

            st = oob_finalize(y, res[0], res[1])
            q.put(("stats", [float(st.degenerate), st.mse, st.response_variance, st.error_pct,
                             st.r_squared, float(st.rows_evaluated)], res[0], res[1]))
        if rank == 0:
            q.put(("forest", gathered))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [10, 7])
def test_two_rank_sharded_fit_equals_single_fit(T):
    col, y = _table()
    p, n = col.shape
    m, mns, seed = 3, 2, 12345
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, m, mns, seed, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict()
    for _ in range(2):
        item = q.get(timeout=120)
        got[item[0]] = item[1:]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    full = Oracle.fit(col, y, n, p, T, m, mns, seed)
    off, f, th, le, ri, va, ib = got["forest"][0]
    assert forests_equal(full, ForestSoA(off, f, th, le, ri, va, inbag=ib)) is None
    stats, rs, rc = Oracle.oob(col, y, n, p, full)
    assert got["stats"][0] == list(stats)
    assert np.array_equal(got["stats"][1].view(np.uint64), rs.view(np.uint64))
    assert np.array_equal(got["stats"][2], rc)


def test_tree_ranges_cover_forest():
    from paper_1811_00156_b200 import shard

    for world in (1, 2, 3, 8):
        for T in (1, 7, 1000):
            rs = [shard.tree_range(r, world, T) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == T
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


GRID_CELLS = [(1, 1), (2, 3), (3, 2), (1, 5), (2, 1)]
GRID_T = [3, 6, 10]


def _grid_compute(cells):
    """Oracle stand-in for grid_oob on one rank: error_pct per (cell, num.trees)."""
    col, y = _table()
    p, n = col.shape
    out = np.zeros((len(cells), len(GRID_T)))
    for i, (m, mns) in enumerate(cells):
        for j, T in enumerate(GRID_T):
            f = Oracle.fit(col, y, n, p, T, m, mns, 777)
            out[i, j] = Oracle.oob(col, y, n, p, f)[0][3]
    return out


def _grid_worker(rank, world, port, q):
    from paper_1811_00156_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = shard.grid_sharded(GRID_CELLS, GRID_T, rank, world, _grid_compute,
                                 shard.torch_allreduce_sum())
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_grid_equals_single_process():
    """C2 sharding (cell i on rank i mod 2) + SUM all-reduce == one process, exactly."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    want = _grid_compute(GRID_CELLS)
    for r in range(2):
        assert np.array_equal(got[r].view(np.uint64), want.view(np.uint64))


def test_cells_and_folds_cover_once():
    from paper_1811_00156_b200 import shard

    for world in (1, 2, 3, 8):
        cells = list(range(37))
        seen = sorted(i for r in range(world) for i, _ in shard.cells_for_rank(cells, r, world))
        assert seen == cells
        fr = [shard.fold_range(r, world, 37) for r in range(world)]
        assert fr[0][0] == 0 and fr[-1][1] == 37
        assert all(a[1] == b[0] for a, b in zip(fr, fr[1:]))


@pytest.mark.parametrize("T,world", [(7, 3), (2, 3)])
def test_gather_forest_ragged_and_empty_shards(T, world):
    """gather_forest over `world` threads (an in-process all_gather on CPU tensors): ragged
    tree ranges, including a rank holding no trees, reassemble the one-shot forest."""
    import threading

    import torch
    from paper_1811_00156_b200 import shard

    col, y = _table()
    p, n = col.shape
    m, mns, seed = 3, 2, 777
    full = Oracle.fit(col, y, n, p, T, m, mns, seed)
    slots, bar = [None] * world, threading.Barrier(world)

    def ag_for(r):
        def ag(lst, t):
            slots[r] = t.clone()
            bar.wait()
            for i in range(world):
                lst[i].copy_(slots[i])
            bar.wait()
        return ag

    got, errs = [None] * world, []

    def run(r):
        try:
            t0, t1 = shard.tree_range(r, world, T)
            if t1 > t0:
                part = Oracle.fit(col, y, n, p, T, m, mns, seed, trees=range(t0, t1))
                off, arrs = part.offsets, (part.feature, part.threshold, part.left, part.value,
                                           part.inbag.reshape(-1).view(np.int32))
            else:
                off = np.zeros(1, np.uint64)
                arrs = (np.zeros(0, np.int32), np.zeros(0), np.zeros(0, np.int32), np.zeros(0),
                        np.zeros(0, np.int32))
            tens = [torch.from_numpy(np.ascontiguousarray(a)) for a in arrs]
            got[r] = shard.gather_forest(off, tens, world, ag_for(r), n)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join(timeout=120)
    assert not errs, errs
    for off, g in got:
        fe, thr, le, va, ib = (t.numpy() for t in g)
        ri = np.where(le < 0, -1, le + 1).astype(np.int32)
        s = ForestSoA(off, fe, thr, le, ri, va, inbag=ib.view(np.uint32).reshape(-1, n))
        assert forests_equal(full, s) is None
