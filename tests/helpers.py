"""Shared test helpers: comparisons and small seeded generators (numpy RNG)."""
import numpy as np

import paper_2507_21253_b200 as B


def same_bits(x: np.ndarray, y: np.ndarray) -> bool:
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def assert_csr_identical(c, o, what=""):
    """row_ptr and col_idx bit-exact, values bit-identical (the reference's
    summation order is reproduced, so no tolerance is needed)."""
    assert c.nrows == o.nrows, what
    assert np.array_equal(np.asarray(c.row_ptr, np.int64), np.asarray(o.row_ptr, np.int64)), \
        f"row_ptr differs {what}"
    assert np.array_equal(np.asarray(c.col_idx), np.asarray(o.col_idx)), f"col_idx differs {what}"
    if not same_bits(c.values, o.values):
        d = np.abs(c.values - o.values) / np.maximum(np.abs(o.values), 1e-300)
        # north-star tolerance: 1e-12 relative; report but demand bitwise.
        raise AssertionError(f"values differ {what}: max rel err {d.max():.3e}, "
                             f"{np.count_nonzero(c.values != o.values)} differ")


def random_csr(nrows, ncols, density, seed, nonnegative=True):
    """Same recipe as reference test_support.hpp:110-122 (Bernoulli pattern,
    values U[0.1,4) or U[-4,4)), drawn from numpy's RNG."""
    rng = np.random.default_rng(seed)
    mask = rng.random((nrows, ncols)) < density
    lo = 0.1 if nonnegative else -4.0
    vals = rng.uniform(lo, 4.0, size=(nrows, ncols))
    r, c = np.nonzero(mask)
    return B.coo_to_csr(nrows, ncols, r, c, vals[r, c])


def identity_csr(n):
    return B.coo_to_csr(n, n, np.arange(n), np.arange(n), np.ones(n))


def csr_from_rows(ncols, rows):
    r = [i for i, cs in enumerate(rows) for _ in cs]
    c = [x for cs in rows for x in cs]
    return B.coo_to_csr(len(rows), ncols, r, c, np.ones(len(c)))


def grouped_identical_rows(groups, k, row_nnz):
    n = max(groups * k, groups * row_nnz)
    r, c = [], []
    for g in range(groups):
        for l in range(k):
            for x in range(row_nnz):
                r.append(g * k + l)
                c.append(g * row_nnz + x)
    return B.coo_to_csr(n, n, r, c, np.ones(len(r)))


def random_assignment(nrows, max_piece, seed):
    rng = np.random.default_rng(seed)
    rows = rng.permutation(nrows)
    out, pos = [], 0
    while pos < nrows:
        take = min(int(rng.integers(1, max(1, max_piece) + 1)), nrows - pos)
        out.append(sorted(rows[pos:pos + take].tolist()))
        pos += take
    return B.ClusterAssignment.from_lists(out)
