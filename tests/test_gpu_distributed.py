"""Multi-GPU data plane on the device.

Only one GPU exists here, and NCCL refuses two ranks on one device, so:
- the engine's own NCCL path (communicator in the handle, B broadcast, row-sharded
  multiply, variable-size all-gather by grouped broadcasts) runs as a world of 1 —
  every code path of bsp_spgemm_rowwise_sharded / bsp_csr_allgather_rows executes,
  with the group of one rank;
- the N = 2 split runs as two processes sharing cuda:0 that exchange over gloo: each
  runs the ENGINE's kernels on its shard (row blocks from bsp_partition_rows; cluster
  runs from bsp_partition_clusters, operand gathered by bsp_csr_select_rows), the
  shards are gathered without padding (distributed.allgather_csr) and rank 0 compares
  the concatenation bit for bit with the single-rank engine result.
The kernels of the two processes never wait on each other (only host-side gloo).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
import paper_2507_21253_b200 as B
from helpers import assert_csr_identical

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_engine_nccl_world_of_one(engine):
    e = B.Engine(0)
    try:
        e.comm_init(1, 0, B.Engine.nccl_unique_id())
        assert e.comm_rank() == (0, 1)
        a = B.make_config(5, 14)
        A, ms = e.broadcast(e.upload(a), 0)
        assert ms >= 0.0
        want = O.spgemm_rowwise(a, a)
        C, info = e.spgemm_rowwise_sharded(A, A, gather=False)
        assert (info["row_begin"], info["row_end"]) == (0, a.nrows)
        assert info["nnz_local"] == want.col_idx.size and info["multiply_ms"] > 0
        assert_csr_identical(C.download(), want, "sharded, one rank")
        G, info = e.spgemm_rowwise_sharded(A, A, gather=True)
        assert_csr_identical(G.download(), want, "sharded + gather, one rank")
        assert_csr_identical(e.allgather_rows(C).download(), want, "allgather_rows, one rank")
    finally:
        e.close()


def test_partition_clusters_and_select_rows(engine):
    a = B.make_config(2, 256)
    A = engine.upload(a)
    asg = engine.hierarchical_clusters(a)
    Ac = engine.build_csr_cluster(A, asg)
    for parts in (1, 2, 3):
        b = engine.partition_clusters(Ac, A, parts)
        assert b[0] == 0 and b[-1] == asg.nclusters and np.all(np.diff(b) >= 0)
    # the split rule on the host mirror (products of each cluster's rows)
    blen = np.diff(a.row_ptr)
    prods = np.array([blen[a.col_idx[a.row_ptr[i]:a.row_ptr[i + 1]]].sum() for i in range(a.nrows)])
    cp = asg.cluster_ptr
    cprod = np.array([prods[asg.rows[cp[c]:cp[c + 1]]].sum() for c in range(asg.nclusters)])
    from paper_2507_21253_b200 import distributed as D
    assert np.array_equal(engine.partition_clusters(Ac, A, 3), D.cluster_split(cprod, 3))
    rows = np.array([5, 0, 5, a.nrows - 1, 17], np.int32)
    S = engine.select_rows(A, rows).download()
    for k, r in enumerate(rows):
        assert np.array_equal(S.row_cols(k), a.row_cols(int(r)))
        assert np.array_equal(S.row_vals(k).view(np.uint64), a.row_vals(int(r)).view(np.uint64))


def _worker(rank, world, port, q):
    import faulthandler
    import sys

    # a hung rank dumps its stacks (stderr) instead of hanging silently
    faulthandler.dump_traceback_later(150, exit=True, file=sys.stderr)
    try:
        _work(rank, world, port, q)
    except BaseException:  # report instead of leaving the peer blocked in gloo
        import traceback

        q.put(("error", rank, traceback.format_exc()))


def _work(rank, world, port, q):
    import datetime

    import torch.distributed as dist
    from paper_2507_21253_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world,
                            timeout=datetime.timedelta(seconds=120))
    try:
        torch.cuda.set_device(0)
        e = B.Engine(0)
        res = {}
        # row shards (R-MAT: heavy rows, windows)
        a = B.make_config(5, 14)
        A = e.upload(a)
        bounds = e.partition_rows(A, A, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        c = e.spgemm_rowwise_range(A, A, r0, r1).download()
        g = D.allgather_csr(torch.from_numpy(c.row_ptr), torch.from_numpy(c.col_idx),
                            torch.from_numpy(c.values))
        if rank == 0:  # compared here: only a small verdict crosses the queue
            assert 0 < bounds[1] < bounds[2]
            assert_csr_identical(
                B.CsrMatrix(a.nrows, a.ncols, g[0].numpy(), g[1].numpy(), g[2].numpy()),
                e.spgemm_rowwise(A, A).download(), "2 row shards")
            res["rows"] = [int(x) for x in bounds]
        # cluster shards (hidden clusters)
        h = B.make_config(2, 256)
        H = e.upload(h)
        asg = e.hierarchical_clusters(h)
        Hc = e.build_csr_cluster(H, asg)
        cb = e.partition_clusters(Hc, H, world)
        Sc, rows, _ = D.cluster_shard(e, H, asg, cb, rank)
        cs = e.spgemm_clusterwise(Sc, H).download()
        g = D.allgather_csr(torch.from_numpy(cs.row_ptr), torch.from_numpy(cs.col_idx),
                            torch.from_numpy(cs.values))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([rows.size], dtype=torch.int64))
        bufs = [torch.zeros(int(s[0]), dtype=torch.int32) for s in sizes]
        for r in range(world):
            t = torch.from_numpy(rows) if r == rank else bufs[r]
            dist.broadcast(t, r)
            bufs[r] = t
        if rank == 0:
            order = torch.cat(bufs).numpy()
            pos = np.empty_like(order)
            pos[order] = np.arange(order.size)
            G = B.CsrMatrix(h.nrows, h.ncols, g[0].numpy(), g[1].numpy(), g[2].numpy())
            # cluster order -> original row order, on the device
            Gd = e.upload(G)
            assert 0 < cb[1] < cb[2]
            assert_csr_identical(e.select_rows(Gd, pos).download(),
                                 e.spgemm_rowwise(H, H).download(), "2 cluster shards")
            res["clusters"] = [int(x) for x in cb]
            q.put(("ok", 0, res))
        e.close()
    finally:
        dist.destroy_process_group()


def test_two_ranks_engine_shards_concatenate_to_the_one_rank_result():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q), daemon=True)
             for r in range(world)]
    for p in procs:
        p.start()
    import faulthandler
    import sys

    faulthandler.dump_traceback_later(200, exit=False, file=sys.stderr)
    try:
        kind, who, res = q.get(timeout=180)
        assert kind == "ok", f"rank {who} failed:\n{res}"
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
    finally:
        faulthandler.cancel_dump_traceback_later()
        for p in procs:
            if p.is_alive():
                p.kill()
    assert res["rows"][1] > 0 and res["clusters"][1] > 0
