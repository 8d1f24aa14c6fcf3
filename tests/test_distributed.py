"""CPU, world_size 2 over gloo: the multi-GPU plumbing of the row-sharded and
cluster-sharded multiply — product-balanced row split, cluster split
snapped to cluster boundaries, B replication by broadcast, per-rank shard multiply
(the oracle stands in for the GPU kernel on CPU; tests/test_gpu_distributed.py runs
the engine's kernels in the shards), global C by a variable-size all-gather (no
padding) — must reproduce the 1-rank C exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import paper_2507_21253_b200 as B
from paper_2507_21253_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if rank == 0:
            a = B.make_config(5, 11)
            meta = torch.tensor([a.nrows, a.nnz()], dtype=torch.int64)
        else:
            a = None
            meta = torch.zeros(2, dtype=torch.int64)
        dist.broadcast(meta, 0)
        n, nnz = (int(x) for x in meta)
        rp = torch.from_numpy(a.row_ptr) if rank == 0 else torch.zeros(n + 1, dtype=torch.int64)
        ci = torch.from_numpy(a.col_idx) if rank == 0 else torch.zeros(nnz, dtype=torch.int32)
        v = torch.from_numpy(a.values) if rank == 0 else torch.zeros(nnz, dtype=torch.float64)
        D.broadcast_csr(rp, ci, v)
        A = O.Csr(n, n, rp.numpy(), ci.numpy(), v.numpy())
        blen = np.diff(A.row_ptr)
        prods = np.array([blen[A.col_idx[A.row_ptr[i]:A.row_ptr[i + 1]]].sum() for i in range(n)])
        bounds = D.product_split(prods, world)
        r0, r1 = D.shard(bounds, rank)
        sub = O.Csr(r1 - r0, n, A.row_ptr[r0:r1 + 1] - A.row_ptr[r0],
                    A.col_idx[A.row_ptr[r0]:A.row_ptr[r1]], A.values[A.row_ptr[r0]:A.row_ptr[r1]])
        c = O.spgemm_rowwise(sub, A)  # stands in for bsp_spgemm_rowwise_range
        grp, gci, gv = D.allgather_csr(torch.from_numpy(c.row_ptr), torch.from_numpy(c.col_idx),
                                       torch.from_numpy(c.values))
        if rank == 0:
            full = O.spgemm_rowwise(A, A)
            ok = (np.array_equal(grp.numpy(), full.row_ptr) and np.array_equal(gci.numpy(), full.col_idx)
                  and np.array_equal(gv.numpy().view(np.uint64), full.values.view(np.uint64)))
            share = [int(prods[bounds[g]:bounds[g + 1]].sum()) for g in range(world)]
            q.put((ok, share, int(prods.sum())))
    finally:
        dist.destroy_process_group()


def test_sharded_multiply_equals_single_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, share, total = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok, "gathered shards differ from the single-rank product"
    assert sum(share) == total and max(share) <= 0.75 * total  # products balanced


def test_product_split_rule():
    prods = np.array([5, 0, 0, 100, 1, 5000, 1, 1, 50, 2, 4097, 3, 70000, 9], dtype=np.int64)
    for parts in (2, 3, 5):
        b = D.product_split(prods, parts)
        assert b[0] == 0 and b[-1] == prods.size and np.all(np.diff(b) >= 0)
        cost = np.array([2 * p if p > 65536 else p for p in prods])
        pre = np.concatenate([[0], np.cumsum(cost)])
        for g in range(1, parts):  # first row whose exclusive cost prefix reaches total*g/parts
            t = cost.sum() * g // parts
            assert pre[b[g]] >= t and (b[g] == 0 or pre[b[g] - 1] < t)




def _cluster_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = B.make_config(2, 128)  # hidden clusters: real multi-member clusters
        cl = O.merge_candidates(a, O.spgemm_topk(a, 7, 0.3), 0.3, 8)
        cp, rows = cl
        blen = np.diff(a.row_ptr)
        prods = np.array([blen[a.col_idx[a.row_ptr[i]:a.row_ptr[i + 1]]].sum()
                          for i in range(a.nrows)])
        cprod = np.array([prods[rows[cp[c]:cp[c + 1]]].sum() for c in range(cp.size - 1)])
        bounds = D.cluster_split(cprod, world)
        c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
        my_rows = rows[cp[c0]:cp[c1]]
        # this rank's clusters (local assignment over its rows, cluster order)
        sub = O.Csr(my_rows.size, a.ncols,
                    np.concatenate([[0], np.cumsum(np.diff(a.row_ptr)[my_rows])]).astype(np.int64),
                    np.concatenate([a.col_idx[a.row_ptr[r]:a.row_ptr[r + 1]] for r in my_rows]),
                    np.concatenate([a.values[a.row_ptr[r]:a.row_ptr[r + 1]] for r in my_rows]))
        lptr = (cp[c0:c1 + 1] - cp[c0]).astype(np.int64)
        c, _, _ = O.spgemm_clusterwise(sub, lptr, np.arange(my_rows.size, dtype=np.int32), a)
        grp, gci, gv = D.allgather_csr(torch.from_numpy(c.row_ptr), torch.from_numpy(c.col_idx),
                                       torch.from_numpy(c.values))
        if rank == 0:
            # rows come back in cluster order: permute to the original row order
            order = rows  # cluster-order position p holds original row rows[p]
            pos = np.empty_like(order)
            pos[order] = np.arange(order.size)
            grp, gci, gv = grp.numpy(), gci.numpy(), gv.numpy()
            lens = np.diff(grp)[pos]
            orp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
            oci = np.concatenate([gci[grp[p]:grp[p + 1]] for p in pos])
            ov = np.concatenate([gv[grp[p]:grp[p + 1]] for p in pos])
            full = O.spgemm_rowwise(a, a)
            ok = (np.array_equal(orp, full.row_ptr) and np.array_equal(oci, full.col_idx)
                  and np.array_equal(ov.view(np.uint64), full.values.view(np.uint64)))
            share = [int(cprod[bounds[g]:bounds[g + 1]].sum()) for g in range(world)]
            q.put((ok, share, int(cprod.sum()), int(bounds[1])))
    finally:
        dist.destroy_process_group()


def test_cluster_sharded_multiply_equals_single_rank():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cluster_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok, share, total, split = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok, "gathered cluster shards differ from the single-rank product"
    assert sum(share) == total and max(share) <= 0.75 * total
    assert 0 < split


def test_cluster_split_rule():
    pc = np.array([5, 0, 7, 100, 1, 50, 1, 1, 50, 2], dtype=np.int64)
    for parts in (2, 3, 4):
        b = D.cluster_split(pc, parts)
        pre = np.concatenate([[0], np.cumsum(pc)])
        assert b[0] == 0 and b[-1] == pc.size and np.all(np.diff(b) >= 0)
        for g in range(1, parts):
            t = pc.sum() * g // parts
            assert pre[b[g]] >= t and (b[g] == 0 or pre[b[g] - 1] < t)
