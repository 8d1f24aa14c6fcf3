"""Host merge (hierarchical clustering, reference clustering.hpp:122-183) timing on
CPU-made candidates: for every column of A, consecutive row pairs sharing it, scored
by Jaccard, up to `k` per row -- the shape of the GPU top-k list (no GPU needed).

usage: python tools/merge_timing.py [--cfg 5] [--lib path/to/libbsp.so] [--dump f.npz]"""
import argparse
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2507_21253_b200 as B


def candidates(a, k=7, seed=1):
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), np.diff(a.row_ptr))
    order = np.lexsort((rows, a.col_idx))
    r, c = rows[order], a.col_idx[order]
    same = c[1:] == c[:-1]
    i, j = r[:-1][same], r[1:][same]
    key = np.unique(np.minimum(i, j) * a.nrows + np.maximum(i, j))
    i, j = key // a.nrows, key % a.nrows
    keep = i != j
    i, j = i[keep], j[keep]
    rng = np.random.default_rng(seed)
    pick = rng.permutation(i.size)[: min(i.size, k * a.nrows)]
    i, j = i[pick], j[pick]
    import scipy.sparse as sp
    m = sp.csr_matrix((np.ones(a.nnz()), a.col_idx, a.row_ptr), shape=(a.nrows, a.ncols))
    deg = np.diff(a.row_ptr)
    sc = np.empty(i.size)
    for s in range(0, i.size, 1 << 20):
        ii, jj = i[s:s + (1 << 20)], j[s:s + (1 << 20)]
        inter = np.asarray(m[ii].multiply(m[jj]).sum(axis=1)).ravel()
        sc[s:s + ii.size] = inter / (deg[ii] + deg[jj] - inter)
    p = np.zeros(i.size, dtype=B.CandidatePair)
    p["i"], p["j"] = i, j
    p["score"] = sc
    return p[sc >= 0.3]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=5)
    ap.add_argument("--scale", type=int, default=None)
    ap.add_argument("--dump", default=None)
    ap.add_argument("--load", default=None)
    args = ap.parse_args()
    a = B.make_config(args.cfg, args.scale)
    if args.load:
        p = np.load(args.load)["p"]
    else:
        p = candidates(a)
        if args.dump:
            np.savez(args.dump, p=p)
    t0 = time.perf_counter()
    asg, trace = B.merge_candidates(a, p)
    dt = time.perf_counter() - t0
    print(f"cfg{args.cfg} n={a.nrows} pairs={p.size} merge_s={dt:.3f} clusters={asg.nclusters} "
          f"merges={trace.size} digest={hashlib.sha1(asg.cluster_ptr.tobytes() + asg.rows.tobytes() + trace.tobytes()).hexdigest()[:16]}")


if __name__ == "__main__":
    main()
