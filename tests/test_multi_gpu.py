"""GPU, world_size 2 (gloo, both ranks on cuda:0): the multi-GPU data path with the REAL
per-rank GPU fits (bench.py --gpus N runs the same code over NCCL, one GPU per rank).

Each rank fits its tree range of the global forest through the C-ABI, the OOB per-row
(sum, count) is chained rank 0 -> 1 on the device (aiwc_oob_accumulate_device; gloo
needs host staging of the send/recv, NCCL does not), and the forest parts are gathered
in rank order.  The result must equal a one-process fit bit for bit (node SoA, in-bag
draws, OOB statistics) -- no kernel of one rank waits on the other's."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, T, q):
    import torch

    import paper_1811_00156_b200 as pkg
    from paper_1811_00156_b200 import shard

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        t = pkg.Table()
        prep = pkg.PreparedDataset.from_table(t, device=0)
        seed = pkg.derive_seed(1, "forest")
        t0, t1 = shard.tree_range(rank, world, T)
        f = pkg.fit(prep, pkg.ForestParams(T, 6, 5, seed), t0, t1, compute_oob_stats=False)
        send, recv = shard.torch_device_transport(host_staging=True)
        res = shard.chained_oob_device(
            t.n, rank, world, torch.device("cuda", 0),
            lambda ps, pc: pkg.oob_accumulate_device(f, prep, ps, pc), send, recv)
        off, fe, th, le, ri, va = f.export()
        ib = f.inbag()
        arrays = [torch.from_numpy(np.ascontiguousarray(a)) for a in
                  (fe, th, le, va, ib.reshape(-1).view(np.int32))]
        goff, g = shard.gather_forest(off, arrays, world, dist.all_gather, t.n)
        if rank == world - 1:
            rs = res[0].cpu().numpy()
            rc = res[1].cpu().numpy().view(np.uint32)
            st = pkg.oob_finalize(t.y, rs, rc)
            q.put(("stats", [st.mse, st.response_variance, st.error_pct, st.r_squared,
                             st.rows_evaluated]))
        if rank == 0:
            q.put(("forest", (goff, *(x.numpy() for x in g))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("T", [90, 33])
def test_two_process_gpu_fit_chain_and_gather(T):
    import paper_1811_00156_b200 as pkg

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, T, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    t = pkg.Table()
    prep = pkg.PreparedDataset.from_table(t)
    full = pkg.fit(prep, pkg.ForestParams(T, 6, 5, pkg.derive_seed(1, "forest")))
    o = full.oob
    assert got["stats"] == [o.mse, o.response_variance, o.error_pct, o.r_squared,
                            o.rows_evaluated]
    goff, fe, th, le, va, ib = got["forest"]
    off, fe1, th1, le1, _, va1 = full.export()
    assert np.array_equal(goff, off)
    assert np.array_equal(fe, fe1) and np.array_equal(le, le1)
    assert np.array_equal(th.view(np.uint64), th1.view(np.uint64))
    assert np.array_equal(va.view(np.uint64), va1.view(np.uint64))
    assert np.array_equal(ib.view(np.uint32).reshape(T, t.n), full.inbag())
