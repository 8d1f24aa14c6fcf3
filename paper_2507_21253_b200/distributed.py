"""Multi-GPU plumbing of the row-sharded SpGEMM.

Rows of C are independent given B, so A is split into contiguous row blocks
balanced by cumulative intermediate products (the split rule of
bsp_partition_rows, include/bsp.h), B is replicated (one broadcast before the
multiply, NCCL over NVLink on GPUs), each rank multiplies its block with no
communication, and C stays sharded.  A global C is assembled only on request
(`allgather_csr`: an all-gather of the shard sizes, then of the padded shard
arrays — NCCL has no all-gather-v).  Everything here works with the NCCL
backend on GPUs and with gloo on CPU tensors (tests/test_distributed.py).
"""
from __future__ import annotations

from typing import Tuple

import numpy as np


def row_cost(row_products: np.ndarray) -> np.ndarray:
    """Partition cost of each row (bsp_partition_rows' rule): a heavy row's
    products (> 4096: planned windows + window symbolic) cost ~2 light ones,
    a hub row's (> 65536) ~3 (per-shard timings, tools/shard_projection.py)."""
    rp = np.asarray(row_products, dtype=np.int64)
    return np.where(rp > 65536, 3 * rp, np.where(rp > 4096, 2 * rp, rp))


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
    """Assemble the global C from per-rank row shards (row_ptr rebased to 0
    on every rank).  Returns (row_ptr, col_idx, values) of the concatenation
    in rank order on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = row_ptr.device
    sizes = torch.tensor([row_ptr.numel() - 1, col_idx.numel()], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes, group=group)
    nrows = [int(s[0]) for s in all_sizes]
    nnzs = [int(s[1]) for s in all_sizes]
    mr, mz = max(nrows), max(max(nnzs), 1)

    def gather(t, length, fill_len):
        buf = torch.zeros(fill_len, dtype=t.dtype, device=dev)
        buf[:length] = t[:length]
        outs = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(outs, buf, group=group)
        return outs

    rps = gather(row_ptr[1:], nrows[dist.get_rank(group)], mr)
    cis = gather(col_idx, nnzs[dist.get_rank(group)], mz)
    vs = gather(values, nnzs[dist.get_rank(group)], mz)
    parts_rp, parts_ci, parts_v = [torch.zeros(1, dtype=row_ptr.dtype, device=dev)], [], []
    off = 0
    for g in range(world):
        parts_rp.append(rps[g][:nrows[g]] + off)
        parts_ci.append(cis[g][:nnzs[g]])
        parts_v.append(vs[g][:nnzs[g]])
        off += nnzs[g]
    return torch.cat(parts_rp), torch.cat(parts_ci), torch.cat(parts_v)
