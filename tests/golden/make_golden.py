"""Generate tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference/proj/include by oracle/Makefile).

The fixtures pin the oracle restatement (oracle/oracle.c) and the host
preprocessing of the product to the reference's own outputs on small seeded
instances of every BASELINE recipe.  Run in the build container:
    python tests/golden/make_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle as O  # noqa: E402
import paper_2507_21253_b200 as B  # noqa: E402

SMALL = {1: 256, 2: 32, 3: 8, 4: 6, 5: 9}
# (cfg, num_frontiers, batch, seed): R-MAT, directed hidden-cluster rows,
# batch > n, a single frontier
FRONTIER_CASES = [(5, 10, 16, 0), (2, 10, 64, 3), (1, 4, 100, 1), (4, 1, 8, 5)]


def main():
    if not O.have_ref():
        O.build(with_ref=True)
    out = {}
    for cfg, sc in SMALL.items():
        a = B.make_config(cfg, sc)
        p = f"cfg{cfg}_"
        out[p + "A_rp"], out[p + "A_ci"], out[p + "A_v"] = a.row_ptr, a.col_idx, a.values
        c = O.ref_spgemm_rowwise(a, a, threads=1)
        out[p + "C_rp"], out[p + "C_ci"], out[p + "C_v"] = c.row_ptr, c.col_idx, c.values
        out[p + "sym"] = O.ref_spgemm_symbolic(a, a, threads=1)
        tk = O.ref_spgemm_topk(a, 7, 0.3, threads=1)
        out[p + "topk_i"], out[p + "topk_j"], out[p + "topk_s"] = tk["i"], tk["j"], tk["score"]
        hp, hr = O.ref_hierarchical_clusters(a, 0.3, 8, threads=1)
        out[p + "hier_ptr"], out[p + "hier_rows"] = hp, hr
        vp, vr = O.ref_variable_length_clusters(a, 0.3, 8)
        out[p + "var_ptr"], out[p + "var_rows"] = vp, vr
        cw, st, slots, colslots = O.ref_spgemm_clusterwise(a, hp, hr, a, threads=1)
        out[p + "cw_stats"] = np.array(st, dtype=np.uint64)
        out[p + "cw_slots"] = np.array([slots, colslots], dtype=np.int64)
        if a.nrows == a.ncols:
            out[p + "rcm"] = O.ref_reorder_rcm(a)
            out[p + "degree"] = O.ref_reorder_degree(a)
    # tall-skinny frontier operands (frontier.hpp:20-77) on the fixtures' A
    for cfg, nf, bt, sd in FRONTIER_CASES:
        p = f"cfg{cfg}_"
        a = O.Csr(len(out[p + "A_rp"]) - 1, len(out[p + "A_rp"]) - 1, out[p + "A_rp"],
                  out[p + "A_ci"], out[p + "A_v"])
        fs = O.ref_generate_frontiers(a, nf, bt, sd)
        q = f"fr_{cfg}_{nf}_{bt}_{sd}_"
        out[q + "count"] = np.array([len(fs)], np.int64)
        for t, f in enumerate(fs):
            out[q + f"{t}_rp"], out[q + f"{t}_ci"] = f.row_ptr, f.col_idx
    for n, seed in [(1, 7), (5, 3), (100, 42), (4096, 4)]:
        out[f"perm_{n}_{seed}"] = O.ref_reorder_random(n, seed)
    path = Path(__file__).with_name("golden.npz")
    np.savez_compressed(path, **out)
    print(path, path.stat().st_size, "bytes,", len(out), "arrays")


if __name__ == "__main__":
    main()
