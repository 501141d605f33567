"""Multi-GPU host logic for the forest path.

Trees shard by global tree index: tree t depends only on (dataset, params, seed, t)
(forest.hpp:182), so rank r grows its own tree range of the global forest and the
union equals a one-GPU fit.  Two exchanges exist:

* OOB (forest.hpp:414-447) sums each row's OOB leaf values in TREE order.  A plain
  all-reduce of per-rank partial sums would reassociate that sum, so it is chained:
  rank r receives the per-row (sum, count) of trees [0, t0_r) from rank r-1, continues
  it with its own trees (aiwc_oob_accumulate), and passes it on; the last rank
  finalises.  Result: bit-identical to the one-GPU / reference value.
* the forest gather (node SoA + in-bag lists) concatenates rank parts in rank order
  (`gather_forest`; `allgather_forest` keeps it on the devices: NCCL all-gather of
  device buffers exported and re-imported through the C-ABI).

The grid search (C2) and hold-one-kernel-out evaluate (C3) shard by cell / fold: each
cell or fold is computed by exactly one rank into a zero-filled array, so a SUM
all-reduce of the arrays combines them exactly (x + 0.0 == x).

The compute is injected (`accumulate(row_sum, row_count)`), so the same logic drives
the GPU path in bench.py (NCCL) and the CPU tests (gloo + the oracle).
"""
from __future__ import annotations

from typing import Callable

import numpy as np


def tree_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Contiguous tree range of `rank` when `total` trees are split over `world` ranks."""
    return (rank * total) // world, ((rank + 1) * total) // world


def _pack(rs: np.ndarray, rc: np.ndarray) -> np.ndarray:
    return np.concatenate([rs.view(np.uint8), rc.astype(np.uint32).view(np.uint8)]).view(np.int32)


def _unpack(buf: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
    raw = buf.view(np.uint8)
    return raw[: 8 * n].view(np.float64).copy(), raw[8 * n: 12 * n].view(np.uint32).copy()


def chained_oob(n: int, rank: int, world: int,
                accumulate: Callable[[np.ndarray, np.ndarray], None],
                send: Callable[[np.ndarray, int], None],
                recv: Callable[[int, int], np.ndarray]):
    """Run the rank chain; returns (row_sum, row_count) on the last rank, else None.

    send(int32_array, dst) / recv(num_int32, src) -> int32_array are the transport
    (torch.distributed send/recv over NCCL or gloo)."""
    if rank > 0:
        rs, rc = _unpack(recv(3 * n, rank - 1), n)
    else:
        rs, rc = np.zeros(n), np.zeros(n, np.uint32)
    accumulate(rs, rc)
    if rank < world - 1:
        send(_pack(rs, rc), rank + 1)
        return None
    return rs, rc


def chained_oob_device(n: int, rank: int, world: int, device,
                       accumulate: Callable[[int, int], None],
                       send: Callable, recv: Callable):
    """The OOB chain with the per-row (sum, count) kept on the GPU: rank r receives the
    device buffers of trees [0, t0_r) from rank r-1 (NCCL send/recv of device tensors,
    or host staging for gloo), continues them in place with its own trees
    (aiwc_oob_accumulate_device) and sends them on.  Returns the device tensors
    (row_sum float64, row_count int32 holding uint32 counts) on the last rank, else None.

    accumulate(d_sum_ptr, d_count_ptr); send(tensor, dst); recv(tensor, src) (in place)."""
    import torch

    rs = torch.zeros(n, dtype=torch.float64, device=device)
    rc = torch.zeros(n, dtype=torch.int32, device=device)
    if rank > 0:
        recv(rs, rank - 1)
        recv(rc, rank - 1)
    if torch.device(device).type == "cuda":
        torch.cuda.current_stream(device).synchronize()
    accumulate(rs.data_ptr(), rc.data_ptr())
    if rank < world - 1:
        send(rs, rank + 1)
        send(rc, rank + 1)
        return None
    return rs, rc


def torch_device_transport(host_staging: bool = False):
    """send / recv of device tensors over the default process group: directly (NCCL over
    NVLink) or through host copies (gloo, the CPU-backend tests)."""
    import torch.distributed as dist

    def send(t, dst: int):
        dist.send(t.cpu() if host_staging else t, dst=dst)

    def recv(t, src: int):
        if host_staging:
            h = t.cpu()
            dist.recv(h, src=src)
            t.copy_(h)
        else:
            dist.recv(t, src=src)

    return send, recv


def torch_transport(device=None):
    """send/recv callables over the default torch.distributed process group."""
    import torch
    import torch.distributed as dist

    def send(arr: np.ndarray, dst: int):
        t = torch.from_numpy(np.ascontiguousarray(arr))
        dist.send(t.to(device) if device is not None else t, dst=dst)

    def recv(count: int, src: int) -> np.ndarray:
        t = torch.empty(count, dtype=torch.int32, device=device)
        dist.recv(t, src=src)
        return t.cpu().numpy()

    return send, recv


def concat_forests(parts):
    """Rank-ordered concatenation of (offsets, feature, threshold, left, right, value,
    inbag) parts into one forest in global tree order."""
    offs, cols = [np.zeros(1, np.uint64)], [[] for _ in range(5)]
    inb = []
    base = np.uint64(0)
    for off, f, th, le, ri, va, ib in parts:
        offs.append(np.asarray(off[1:], np.uint64) + base)
        base += np.uint64(off[-1])
        for k, a in enumerate((f, th, le, ri, va)):
            cols[k].append(a)
        inb.append(ib)
    return (np.concatenate(offs), *[np.concatenate(c) for c in cols],
            np.concatenate(inb) if inb and inb[0] is not None else None)


def gather_forest(off_local, arrays, world: int, all_gather, n: int = 0):
    """All-gather of the tree-seed shards of a forest: every rank ends with the
    whole forest in global tree order (rank order = tree order, `tree_range`).

    off_local: this rank's host offsets (trees_local + 1).  arrays: this rank's flat
    tensors [feature i32, threshold f64, left i32, value f64], plus the in-bag draws
    (trees_local x n, int32 view of u32) when n > 0, all on the collective's device.
    all_gather(list_of_tensors, tensor) is torch.distributed.all_gather (NCCL over NVLink
    on the GPUs, gloo in the CPU tests).  Ragged shards are padded to the largest.
    Returns (offsets u64 host, [gathered tensors in the same order])."""
    import torch

    dev = arrays[0].device
    off_local = np.asarray(off_local, np.uint64)
    counts = np.diff(off_local).astype(np.int64)
    meta = torch.tensor([len(counts), int(off_local[-1])], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    all_gather(metas, meta)
    metas = [(int(m[0]), int(m[1])) for m in (x.cpu().numpy() for x in metas)]
    tmax = max(m[0] for m in metas)
    nmax = max(m[1] for m in metas)
    ct = torch.zeros(max(1, tmax), dtype=torch.int64, device=dev)
    ct[:len(counts)] = torch.from_numpy(counts).to(dev)
    cts = [torch.empty_like(ct) for _ in range(world)]
    all_gather(cts, ct)
    all_counts = np.concatenate([c.cpu().numpy()[:m[0]] for c, m in zip(cts, metas)])
    offsets = np.zeros(len(all_counts) + 1, np.uint64)
    offsets[1:] = np.cumsum(all_counts).astype(np.uint64)
    out = []
    for k, a in enumerate(arrays):
        node_array = k < 4  # nodes: N_r entries; in-bag: T_r x n
        size = max(1, nmax if node_array else tmax * n)
        buf = torch.zeros(size, dtype=a.dtype, device=dev)
        buf[:a.numel()] = a
        parts = [torch.empty_like(buf) for _ in range(world)]
        all_gather(parts, buf)
        out.append(torch.cat([q[:(m[1] if node_array else m[0] * n)]
                              for q, m in zip(parts, metas)]))
        del parts, buf
    return offsets, out


def host_staged_all_gather(all_gather):
    """all_gather of device tensors through host copies (gloo)."""
    def ag(outs, t):
        h = [o.cpu() for o in outs]
        all_gather(h, t.cpu())
        for o, x in zip(outs, h):
            o.copy_(x)
    return ag


def allgather_forest(forest, world: int, device: int, all_gather=None, with_inbag=False):
    """Device path of `gather_forest`: the local shard is copied device-to-device out of
    the fitted forest (aiwc_forest_export_device), all-gathered over NCCL, and the whole
    forest is rebuilt on the device (aiwc_forest_import_device) — no host round trip."""
    import torch

    from . import Forest

    if all_gather is None:
        import torch.distributed as dist

        all_gather = dist.all_gather
    dev = torch.device("cuda", device)
    N, T, n = forest.total_nodes, forest.num_trees, forest.n
    fe = torch.empty(N, dtype=torch.int32, device=dev)
    th = torch.empty(N, dtype=torch.float64, device=dev)
    le = torch.empty(N, dtype=torch.int32, device=dev)
    va = torch.empty(N, dtype=torch.float64, device=dev)
    arrays = [fe, th, le, va]
    ib = None
    if with_inbag:
        ib = torch.empty(T * n, dtype=torch.int32, device=dev)
        arrays.append(ib)
    torch.cuda.synchronize(dev)
    forest.export_device(fe.data_ptr(), th.data_ptr(), le.data_ptr(), va.data_ptr(),
                         ib.data_ptr() if ib is not None else None)
    off, out = gather_forest(forest.offsets(), arrays, world, all_gather,
                             n if with_inbag else 0)
    torch.cuda.synchronize(dev)
    return Forest.from_device(off, *(t.data_ptr() for t in out[:4]),
                              out[4].data_ptr() if with_inbag else None,
                              n if with_inbag else 0, device)


def cells_for_rank(cells, rank: int, world: int):
    """Round-robin share of grid cells (cell i goes to rank i mod G):
    returns [(index, cell)] for this rank."""
    return [(i, c) for i, c in enumerate(cells) if i % world == rank]


def fold_range(rank: int, world: int, folds: int) -> tuple[int, int]:
    """Contiguous fold range of `rank` for a sharded evaluate."""
    return tree_range(rank, world, folds)


def grid_sharded(cells, tree_counts, rank: int, world: int,
                 compute: Callable[[list], np.ndarray],
                 allreduce_sum: Callable[[np.ndarray], np.ndarray]) -> np.ndarray:
    """Grid objective over all ranks: rank r computes its round-robin cells with
    `compute(list_of_cells) -> [k, len(tree_counts)]`, the per-rank results are placed
    in a zero-filled [len(cells), len(tree_counts)] array and summed over ranks."""
    mine = cells_for_rank(cells, rank, world)
    out = np.zeros((len(cells), len(tree_counts)))
    if mine:
        res = compute([c for _, c in mine])
        for j, (i, _) in enumerate(mine):
            out[i] = res[j]
    return allreduce_sum(out)


def torch_allreduce_sum(device=None):
    """SUM all-reduce of a float64 numpy array over the default process group."""
    import torch
    import torch.distributed as dist

    def f(a: np.ndarray) -> np.ndarray:
        t = torch.from_numpy(np.ascontiguousarray(a, np.float64))
        t = t.to(device) if device is not None else t
        dist.all_reduce(t)
        return t.cpu().numpy()

    return f
