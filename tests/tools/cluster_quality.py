"""cfg2 (hidden clusters) clustering quality and cluster-wise vs row-wise timing.

SURVEY 8(c) (iii)/(iv): minhash/LSH (the north-star GPU candidate step, not in the
reference) has no oracle, so it is judged by
  - recovery of cfg2's planted template groups (a group = the 8 child rows of one
    template; recovered = some cluster has exactly those rows) and purity (clusters
    whose rows all come from one template), against the reference's own top-k
    hierarchical clustering bar (97.11 % recovered, 100 % pure on the survey probe);
  - C parity (cluster-wise C == row-wise C bit for bit, whatever the clustering);
  - time of the candidate step and of the multiply it enables.
The planted group of each (permuted) row is recovered by permuting an identity
matrix with the generator's own row permutation (reorder_random(n, perm_seed)).

usage: python tests/tools/cluster_quality.py [--scale NT] [--steps K] [--ref]  (one JSON line)
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch

import paper_2507_21253_b200 as B


def planted_groups(cfg):
    """template id of every row of the generated (row-permuted) cfg2 matrix."""
    nt, ch = cfg["ntemplates"], cfg["children"]
    n = nt * ch
    eye = B.coo_to_csr(n, n, np.arange(n), np.arange(n), np.ones(n))
    perm = B.reorder_random(n, cfg["perm_seed"])
    moved = B.permute_rows(eye, perm)  # row i of the result = old row col_idx[i]
    return moved.col_idx.astype(np.int64) // ch


def quality(asg, tmpl, children):
    cp, rows = asg.cluster_ptr, asg.rows
    sizes = np.diff(cp)
    cid = np.repeat(np.arange(cp.size - 1), sizes)
    t_of = tmpl[rows]
    # purity: every row of a cluster from one template
    first = t_of[cp[:-1]]
    pure = np.ones(cp.size - 1, bool)
    np.logical_and.at(pure, cid, t_of == first[cid])
    # exact recovery: a cluster of `children` rows, pure, and its template has exactly
    # those rows (templates have `children` rows each)
    exact = pure & (sizes == children)
    nt = int(tmpl.max()) + 1
    hist = np.bincount(sizes, minlength=children + 1)
    return {"clusters": int(cp.size - 1), "recovered": int(exact.sum()), "templates": nt,
            "recovered_pct": 100.0 * exact.sum() / nt, "pure_pct": 100.0 * pure.mean(),
            "size_hist": {int(k): int(v) for k, v in enumerate(hist) if v}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=None, help="templates (default: cfg2's 32768)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--ref", action="store_true", help="also the reference's CPU clustering")
    args = ap.parse_args()
    cfg = dict(B.CONFIGS[2])
    if args.scale:
        cfg["ntemplates"] = args.scale
    a = B.make_config(2, args.scale)
    tmpl = planted_groups(cfg)
    torch.cuda.set_device(0)
    eng = B.Engine(0)
    st = torch.cuda.Stream()
    eng.set_stream(st.cuda_stream)
    A = eng.upload(a)
    products = eng.spgemm_products(A, A)

    def timed(fn, steps=args.steps):
        for _ in range(2):
            fn().free()
        torch.cuda.synchronize()
        ts = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            C = fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
            C.free()
        return {"best_ms": min(ts), "mean_ms": float(np.mean(ts)),
                "gflops": 2 * products / min(ts) / 1e6}

    out = {"cfg": "cfg2", "n": a.nrows, "nnz_a": a.nnz(), "products": products}
    row = timed(lambda: eng.spgemm_rowwise(A, A))
    out["rowwise"] = row
    want = eng.spgemm_rowwise(A, A).download()
    rs = eng.rowwise_access_stats(A, A)
    out["rowwise_b_row_loads"] = int(rs.b_row_loads)
    for method in ("topk", "minhash"):
        t0 = time.perf_counter()
        asg = eng.hierarchical_clusters(a, method=method, nhash=64)
        tc = time.perf_counter() - t0
        q = quality(asg, tmpl, cfg["children"])
        Ac = eng.build_csr_cluster(A, asg)
        got = eng.spgemm_clusterwise(Ac, A).download()
        exact = (np.array_equal(got.row_ptr, want.row_ptr) and
                 np.array_equal(got.col_idx, want.col_idx) and
                 np.array_equal(got.values.view(np.uint64), want.values.view(np.uint64)))
        cl = timed(lambda: eng.spgemm_clusterwise(Ac, A))
        acs = eng.cluster_access_stats(Ac, A)
        out[method] = dict(q, clustering_s=tc, clusterwise=cl, c_bit_identical=bool(exact),
                           speedup_vs_rowwise=row["best_ms"] / cl["best_ms"],
                           b_row_loads=int(acs.b_row_loads),
                           b_row_load_reduction=rs.b_row_loads / max(1, acs.b_row_loads))
    if args.ref:
        import oracle as O

        t0 = time.perf_counter()
        cp, rows = O.ref_hierarchical_clusters(a)
        tr = time.perf_counter() - t0
        ra = B.ClusterAssignment(cp, rows)
        acs = eng.cluster_access_stats(eng.build_csr_cluster(A, ra), A)
        out["reference_topk"] = dict(quality(ra, tmpl, cfg["children"]), clustering_s=tr,
                                     threads=os.cpu_count(), b_row_loads=int(acs.b_row_loads),
                                     b_row_load_reduction=rs.b_row_loads / max(1, acs.b_row_loads))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
