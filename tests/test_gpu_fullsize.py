"""Parity at BASELINE.json's full sizes.

The oracle finishes cfg1 and cfg2 at full size in seconds, so those are compared
bit-for-bit (test_gpu_rowwise covers cfg1 at full size; cfg2 is here, row-wise and
cluster-wise).  cfg3 (C ~285 GB, in 4 row ranges), cfg4 (1.5e9 products) and cfg5
(1.2e10 products, 138 GB of C) are checked on the device through size-independent properties of C = A·A:

- structure: row_ptr starts at 0, is non-decreasing, ends at nnz(C), and every
  row's length equals the symbolic pass's count; the number of products equals
  the pinned count of the seeded recipe;
- sortedness: column indices strictly increase inside every row and lie in
  [0, ncols) (the reference's sorted, duplicate-free rows, spgemm.hpp:98-104);
- linearity: C·x = A·(A·x) for a seeded x in [0, 1).  All values of these
  recipes are >= 0 except cfg4's off-diagonal -1, so the bound is taken against
  |C|·|x|: |C·x - A·(A·x)| <= 1e-9 · (|C|·|x|) entrywise (fp64, summation
  orders differ between the two sides; the kernels themselves are bit-exact).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2507_21253_b200 as B
from helpers import assert_csr_identical

pytestmark = pytest.mark.gpu

RTOL = 1e-9
CHUNK = 1 << 28  # entries of C per property chunk (2 GB of fp64 temporaries)


class _Cai:
    """Zero-copy device view of an engine-owned buffer (__cuda_array_interface__)."""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


def _view(ptr, n, typestr):
    return torch.as_tensor(_Cai(ptr, n, typestr), device="cuda")


def _spmv(rp, ci, v, x, absval=False):
    """y = M·x for a device CSR (row_ptr int64, col int32, fp64), in row chunks."""
    n = rp.numel() - 1
    y = torch.zeros(n, dtype=torch.float64, device=x.device)
    rph = rp.cpu().numpy()
    r0 = 0
    while r0 < n:
        r1 = int(np.searchsorted(rph, rph[r0] + CHUNK, side="right")) - 1
        r1 = min(n, max(r1, r0 + 1))
        s, e = int(rph[r0]), int(rph[r1])
        if e > s:
            vals = v[s:e].abs() if absval else v[s:e]
            prod = vals * x[ci[s:e].long()]
            rows = torch.repeat_interleave(torch.arange(r0, r1, device=x.device),
                                           rp[r0 + 1:r1 + 1] - rp[r0:r1])
            y.index_add_(0, rows, prod)
        r0 = r1
    return y


def _check_properties(engine, a, pinned_products, nchunks=1):
    """C = A·A in `nchunks` row ranges (bsp_spgemm_rowwise_range, the cost split of
    bsp_partition_rows), each checked and freed before the next (cfg3's C is 285 GB)."""
    dev = torch.device("cuda")
    rpA = torch.from_numpy(a.row_ptr).to(dev)
    ciA = torch.from_numpy(a.col_idx).to(dev)
    vA = torch.from_numpy(a.values).to(dev)
    torch.cuda.synchronize()  # the engine runs on its own stream
    A = engine.view_torch(a.nrows, a.ncols, rpA, ciA, vA)
    assert engine.spgemm_products(A, A) == pinned_products
    cnt = torch.from_numpy(engine.spgemm_symbolic(A, A)).to(dev)
    g = torch.Generator(device=dev).manual_seed(2507)
    x = torch.rand(a.ncols, dtype=torch.float64, device=dev, generator=g)
    z = _spmv(rpA, ciA, vA, _spmv(rpA, ciA, vA, x))
    bounds = ([0, a.nrows] if nchunks == 1
              else [int(b) for b in engine.partition_rows(A, A, nchunks)])
    total = 0
    for r0, r1 in zip(bounds[:-1], bounds[1:]):
        Cd = (engine.spgemm_rowwise(A, A) if nchunks == 1
              else engine.spgemm_rowwise_range(A, A, r0, r1))
        engine.synchronize()
        try:
            n, nnz = Cd.nrows, Cd.nnz()
            assert n == r1 - r0
            total += nnz
            if nnz == 0:
                assert int(cnt[r0:r1].sum()) == 0
                continue
            rp = _view(Cd.s.row_ptr, n + 1, "<i8")
            ci = _view(Cd.s.col_idx, nnz, "<i4")
            v = _view(Cd.s.values, nnz, "<f8")
            # structure
            assert int(rp[0]) == 0 and int(rp[-1]) == nnz
            assert bool(((rp[1:] - rp[:-1]) >= 0).all())
            assert torch.equal(rp[1:] - rp[:-1], cnt[r0:r1])
            # sortedness, chunk by chunk (a chunk boundary inside a row is
            # checked by overlapping chunks by one entry)
            for s in range(0, nnz, CHUNK):
                e = min(nnz, s + CHUNK + 1)
                c = ci[s:e]
                assert int(c.min()) >= 0 and int(c.max()) < a.ncols
                starts = torch.zeros(e - s, dtype=torch.bool, device=dev)
                lo = int(torch.searchsorted(rp, torch.tensor([s], device=dev), right=True)[0])
                hi = int(torch.searchsorted(rp, torch.tensor([e - 1], device=dev), right=True)[0])
                rs = rp[lo:hi] - s  # row starts inside (s, e)
                starts[rs[(rs > 0) & (rs < e - s)]] = True
                assert bool(((c[1:] > c[:-1]) | starts[1:]).all()), f"unsorted near entry {s}"
            # linearity
            cx = _spmv(rp, ci, v, x)
            bound = _spmv(rp, ci, v, x, absval=True)
            worst = float(((cx - z[r0:r1]).abs() - RTOL * bound).max())
            assert worst <= 0.0, f"rows [{r0},{r1}) C·x vs A·(A·x): max excess {worst}"
        finally:
            Cd.free()
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
    return total


def test_cfg2_full_rowwise_and_clusterwise_bit_exact(engine):
    """cfg2 at its BASELINE size (n = 262144), both entry points vs the oracle."""
    a = B.make_config(2)
    o = O.spgemm_rowwise(a, a)
    A = engine.upload(a)
    assert_csr_identical(engine.spgemm_rowwise(A, A).download(), o, "cfg2 full row-wise")
    asg = engine.hierarchical_clusters(a)
    Ac = engine.build_csr_cluster(A, asg)
    assert_csr_identical(engine.spgemm_clusterwise(Ac, A).download(), o, "cfg2 full cluster-wise")


def test_cfg4_full_properties(engine):
    """27-point stencil 128^3 (n = 2097152, randomly permuted), C = A·A."""
    a = B.make_config(4)
    p = int(np.sum(np.diff(a.row_ptr)[a.col_idx]))  # sum over A's entries of B's row lengths
    _check_properties(engine, a, p)


def test_cfg5_full_properties(engine):
    """R-MAT 22 ef 8 (the bench workload): 11,943,554,182 products, 138 GB of C."""
    a = B.make_config(5)
    assert _check_properties(engine, a, 11943554182) == 11522129996


def test_cfg3_full_properties_row_chunks(engine):
    """R-MAT 20 ef 16 (n = 1048576): C (~285 GB) exceeds HBM, so it is produced and
    checked in 4 row ranges of equal product cost, as the e2e path and cfg3 runs do."""
    a = B.make_config(3)
    p = int(np.sum(np.diff(a.row_ptr)[a.col_idx]))
    _check_properties(engine, a, p, nchunks=4)
