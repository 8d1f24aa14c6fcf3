"""Multi-GPU plumbing of the row-sharded SpGEMM.

Rows of C are independent given B, so A is split into contiguous row blocks
balanced by cumulative intermediate products (the split rule of
bsp_partition_rows, include/bsp.h), B is replicated (one broadcast before the
multiply, NCCL over NVLink on GPUs), each rank multiplies its block with no
communication, and C stays sharded.  A global C is assembled only on request
(`allgather_csr`: an all-gather of the shard sizes, then one broadcast per rank
of its exact arrays — NCCL has no all-gather-v; no padding).  The engine does
the same on device memory with its own NCCL communicator
(Engine.comm_init / spgemm_rowwise_sharded / allgather_rows); the helpers here
mirror its rules for torch.distributed callers and the gloo CPU tests
(tests/test_distributed.py).  Cluster-wise shards split at cluster boundaries
(cluster_split / cluster_shard).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def row_cost(row_products: np.ndarray) -> np.ndarray:
    """Partition cost of each row (bsp_partition_rows' rule): a hub row's products
    (> 65536 per row) cost ~2x the others' (fitted to per-shard timings,
    tools/shard_projection.py: 21.2 / 19.7 / 40.7 ms per 1e9 products of light /
    windowed / hub rows)."""
    rp = np.asarray(row_products, dtype=np.int64)
    return np.where(rp > 65536, 2 * rp, rp)


def product_split(row_products: np.ndarray, nparts: int) -> np.ndarray:
    """Bounds b[0..nparts] with b[g] = first row whose exclusive cost prefix
    reaches total*g/nparts (cost = row_cost); monotone, b[0]=0,
    b[-1]=nrows; identical to the rule of bsp_partition_rows."""
    n = int(row_products.size)
    cost = row_cost(row_products)
    pre = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cost, out=pre[1:])
    total = int(pre[-1])
    b = np.zeros(nparts + 1, dtype=np.int64)
    for g in range(1, nparts):
        target = (total * g) // nparts
        r = int(np.searchsorted(pre, target, side="left"))
        b[g] = max(b[g - 1], min(r, n))
    b[nparts] = n
    return b


def shard(bounds: np.ndarray, rank: int) -> Tuple[int, int]:
    return int(bounds[rank]), int(bounds[rank + 1])


def broadcast_csr(row_ptr, col_idx, values, src: int = 0, group=None):
    """Replicate a CSR held by `src` (tensors already sized on every rank)."""
    import torch.distributed as dist

    for t in (row_ptr, col_idx, values):
        dist.broadcast(t, src, group=group)


def allgather_csr(row_ptr, col_idx, values, group=None):
    """Assemble the global C from per-rank row shards (row_ptr rebased to 0 on
    every rank), in rank order, on every rank: an all-gather of the shard sizes,
    then one broadcast per rank of its exact arrays — no padding (NCCL has no
    all-gather-v; the engine's bsp_csr_allgather_rows does the same with grouped
    NCCL broadcasts on device memory).  Works on CPU tensors with gloo."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    me = dist.get_rank(group)
    dev = row_ptr.device
    sizes = torch.tensor([row_ptr.numel() - 1, col_idx.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    nrows = [int(x[0]) for x in all_sizes]
    nnzs = [int(x[1]) for x in all_sizes]
    rp = torch.zeros(sum(nrows) + 1, dtype=row_ptr.dtype, device=dev)
    ci = torch.empty(sum(nnzs), dtype=col_idx.dtype, device=dev)
    v = torch.empty(sum(nnzs), dtype=values.dtype, device=dev)
    r_off = z_off = 0
    for g in range(world):
        seg_rp = rp[1 + r_off:1 + r_off + nrows[g]]
        seg_ci = ci[z_off:z_off + nnzs[g]]
        seg_v = v[z_off:z_off + nnzs[g]]
        if g == me:
            seg_rp.copy_(row_ptr[1:])
            seg_ci.copy_(col_idx)
            seg_v.copy_(values)
        for t in (seg_rp, seg_ci, seg_v):
            if t.numel():
                buf = t.contiguous()
                dist.broadcast(buf, g, group=group)
                t.copy_(buf)
        seg_rp += z_off
        r_off += nrows[g]
        z_off += nnzs[g]
    return rp, ci, v


def cluster_split(cluster_products: np.ndarray, nparts: int) -> np.ndarray:
    """Cluster-boundary split (bsp_partition_clusters' rule): bounds over clusters,
    b[g] = the first cluster whose exclusive product prefix reaches total*g/nparts."""
    pc = np.asarray(cluster_products, dtype=np.int64)
    pre = np.zeros(pc.size + 1, dtype=np.int64)
    np.cumsum(pc, out=pre[1:])
    b = np.zeros(nparts + 1, dtype=np.int64)
    for g in range(1, nparts):
        c = int(np.searchsorted(pre, (int(pre[-1]) * g) // nparts, side="left"))
        b[g] = max(b[g - 1], min(c, pc.size))
    b[nparts] = pc.size
    return b


def cluster_shard(engine, A, asg, bounds, rank):
    """This rank's cluster-wise operand: the clusters [bounds[rank], bounds[rank+1])
    of `asg` (a ClusterAssignment of A), their rows gathered on the device in cluster
    order (bsp_csr_select_rows) and formatted as CSR_Cluster over those rows.
    Returns (DeviceCsrCluster, rows): C = spgemm_clusterwise(shard, B) has one row
    per entry of `rows` (original row ids, cluster order)."""
    from . import ClusterAssignment

    c0, c1 = int(bounds[rank]), int(bounds[rank + 1])
    cp = asg.cluster_ptr
    rows = asg.rows[cp[c0]:cp[c1]].astype(np.int32)
    A_sub = engine.select_rows(A, rows)
    local = ClusterAssignment(cp[c0:c1 + 1] - cp[c0], np.arange(rows.size, dtype=np.int32))
    return engine.build_csr_cluster(A_sub, local), rows, A_sub
