"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the SpGEMM path.

Two checkers, both used only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs (never by the product):

* ``liboracle.so`` — oracle.c, a plain-C restatement of the reference
  algorithms (each function cites reference file:line);
* ``_ref/libcspgemm_ref.so`` — the UNMODIFIED reference headers from
  /root/reference/proj/include compiled by oracle/Makefile (present wherever
  it was built; it travels to the GPU box with the snapshot).

The restatement is pinned against the reference build and against the
golden vectors in tests/golden/ (see tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from collections import namedtuple
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libcspgemm_ref.so"
REF_INCLUDE = Path("/root/reference/proj/include")

Csr = namedtuple("Csr", "nrows ncols row_ptr col_idx values")

i32, i64, u64, dbl = C.c_int32, C.c_int64, C.c_uint64, C.c_double
vp = C.c_void_p
P = C.POINTER


class orc_candidate(C.Structure):
    _fields_ = [("i", i32), ("j", i32), ("score", dbl)]


class orc_access_stats(C.Structure):
    _fields_ = [("b_row_loads", u64), ("a_inner_iters", u64), ("placeholder_skips", u64)]


class orc_cluster(C.Structure):
    _fields_ = [("nclusters", i64), ("nrows", i64), ("ncols", i64), ("ncolslots", i64),
                ("nslots", i64), ("cluster_sizes", P(i32)), ("cluster_col_ptr", P(i64)),
                ("col_idx", P(i32)), ("value_ptr", P(i64)), ("values", P(dbl)),
                ("valid", P(u64)), ("row_map", P(i32))]


CAND = np.dtype([("i", np.int32), ("j", np.int32), ("score", np.float64)])

_orc = None
_ref = None


def build(with_ref: bool = True) -> None:
    """Build liboracle.so (and oracle/_ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", str(HERE), "all"], check=True)
    if with_ref and REF_INCLUDE.exists():
        subprocess.run(["make", "-s", "-C", str(HERE), "ref"], check=True)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build(with_ref=False)
        l = C.CDLL(str(ORACLE_SO))
        l.orc_spgemm_symbolic.argtypes = [i64, i64, vp, vp, vp, vp, vp]
        l.orc_spgemm_rowwise.argtypes = [i64, i64, vp, vp, vp, vp, vp, vp, vp, P(P(i32)), P(P(dbl))]
        l.orc_spgemm_rowwise.restype = i64
        l.orc_jaccard.argtypes = [vp, vp, i64, i64]
        l.orc_jaccard.restype = dbl
        l.orc_spgemm_topk.argtypes = [i64, vp, vp, vp, vp, i32, dbl, P(P(orc_candidate))]
        l.orc_spgemm_topk.restype = i64
        l.orc_build_csr_cluster.argtypes = [i64, i64, vp, vp, vp, i64, vp, vp, P(orc_cluster)]
        l.orc_cluster_to_csr.argtypes = [P(orc_cluster), vp, P(P(i32)), P(P(dbl))]
        l.orc_cluster_to_csr.restype = i64
        l.orc_spgemm_clusterwise.argtypes = [P(orc_cluster), i64, vp, vp, vp, P(orc_cluster),
                                             P(orc_access_stats)]
        l.orc_cluster_free.argtypes = [P(orc_cluster)]
        l.orc_merge_candidates.argtypes = [i64, vp, vp, vp, i64, dbl, i32, vp]
        l.orc_merge_candidates.restype = i64
        l.orc_free.argtypes = [vp]
        l.orc_gen_rmat.argtypes = [i32, i32, dbl, dbl, dbl, u64, P(i64), P(P(i64)), P(P(i32)),
                                   P(P(dbl))]
        _orc = l
    return _orc


def have_ref() -> bool:
    return REF_SO.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError("oracle/_ref not built (needs /root/reference; run make -C oracle ref)")
        l = C.CDLL(str(REF_SO))
        l.ref_last_error.restype = C.c_char_p
        l.ref_spgemm_rowwise.argtypes = [i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i64, i64, C.c_int,
                                         P(i64), P(P(i64)), P(P(i32)), P(P(dbl))]
        l.ref_spgemm_symbolic.argtypes = [i64, i64, vp, vp, i64, i64, vp, vp, C.c_int, vp]
        l.ref_spgemm_topk.argtypes = [i64, i64, vp, vp, i32, dbl, C.c_int, P(i64),
                                      P(P(orc_candidate))]
        l.ref_hierarchical_clusters.argtypes = [i64, i64, vp, vp, dbl, i32, C.c_int, P(i64),
                                                P(P(i64)), P(P(i32))]
        l.ref_variable_length_clusters.argtypes = [i64, i64, vp, vp, dbl, i32, P(i64), P(P(i64)),
                                                   P(P(i32))]
        l.ref_spgemm_clusterwise.argtypes = [i64, i64, vp, vp, vp, i64, i64, vp, vp, vp, i64, vp, vp,
                                             C.c_int, P(i64), P(P(i64)), P(P(i32)), P(P(dbl)),
                                             vp, P(i64), P(i64)]
        l.ref_time_clusterwise.argtypes = [i64, i64, vp, vp, vp, i64, vp, vp, C.c_int, C.c_int,
                                           P(dbl)]
        l.ref_reorder_rcm.argtypes = [i64, i64, vp, vp, vp]
        l.ref_reorder_random.argtypes = [i64, u64, vp]
        l.ref_reorder_degree.argtypes = [i64, i64, vp, vp, vp]
        l.ref_permute_symmetric.argtypes = [i64, i64, vp, vp, vp, vp, P(P(i64)), P(P(i32)),
                                            P(P(dbl))]
        l.ref_jaccard.argtypes = [i64, i64, vp, vp, i64, i64, P(dbl)]
        l.ref_generate_frontiers.argtypes = [i64, i64, vp, vp, i64, i64, u64, P(i64), P(i64),
                                             P(P(i64)), P(P(i64)), P(P(i32))]
        l.ref_free.argtypes = [vp]
        l.ref_load_matrix_market.argtypes = [C.c_char_p, P(i64), P(i64), P(i64), P(P(i64)),
                                             P(P(i32)), P(P(dbl))]
        l.ref_load_permutation.argtypes = [C.c_char_p, i64, vp]
        l.ref_write_matrix_market.argtypes = [i64, i64, vp, vp, vp, C.c_char_p]
        l.ref_fmt_double.argtypes = [dbl, C.c_char_p, C.c_int]
        l.ref_bench_csv_row.argtypes = [C.c_char_p, C.c_int, C.c_int, u64, C.c_char_p, C.c_int,
                                        dbl, C.c_int, C.c_int, C.c_int, C.c_int, u64, C.c_int,
                                        C.c_int, C.c_int, vp, vp, dbl, dbl, C.c_char_p, C.c_int]
        l.ref_csr_new.argtypes = [i64, i64, vp, vp, vp]
        l.ref_csr_new.restype = vp
        l.ref_csr_delete.argtypes = [vp]
        l.ref_time_rowwise.argtypes = [vp, vp, C.c_int, P(dbl), P(i64)]
        l.ref_cluster_new.argtypes = [vp, i64, vp, vp]
        l.ref_cluster_new.restype = vp
        l.ref_cluster_delete.argtypes = [vp]
        l.ref_time_clusterwise_prepared.argtypes = [vp, vp, C.c_int, P(dbl), P(i64)]
        _ref = l
    return _ref


def _arr(ptr, n, dtype, free):
    out = np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0, dtype)
    free(C.cast(ptr, vp))
    return out.astype(dtype, copy=False)


def _csr_args(a):
    return (np.ascontiguousarray(a.row_ptr, np.int64), np.ascontiguousarray(a.col_idx, np.int32),
            np.ascontiguousarray(a.values, np.float64))


# ---------------------------------------------------------------- restatement
def spgemm_symbolic(a, b) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    brp, bci, _ = _csr_args(b)
    out = np.zeros(a.nrows, np.int64)
    lib().orc_spgemm_symbolic(a.nrows, b.ncols, _p(arp), _p(aci), _p(brp), _p(bci), _p(out))
    return out


def spgemm_rowwise(a, b) -> Csr:
    arp, aci, av = _csr_args(a)
    brp, bci, bv = _csr_args(b)
    crp = np.zeros(a.nrows + 1, np.int64)
    cc, cv = P(i32)(), P(dbl)()
    nnz = lib().orc_spgemm_rowwise(a.nrows, b.ncols, _p(arp), _p(aci), _p(av), _p(brp), _p(bci),
                                   _p(bv), _p(crp), C.byref(cc), C.byref(cv))
    return Csr(a.nrows, b.ncols, crp, _arr(cc, nnz, np.int32, lib().orc_free),
               _arr(cv, nnz, np.float64, lib().orc_free))


def transpose_pattern(a):
    """Pattern transpose (stable; rows sorted) in numpy."""
    rows = np.repeat(np.arange(a.nrows, dtype=np.int64), np.diff(a.row_ptr))
    order = np.lexsort((rows, a.col_idx))
    cols_t = rows[order].astype(np.int32)
    cnt = np.bincount(a.col_idx, minlength=a.ncols)
    rp = np.zeros(a.ncols + 1, np.int64)
    rp[1:] = np.cumsum(cnt)
    return Csr(a.ncols, a.nrows, rp, cols_t, np.ones(cols_t.size))


def spgemm_topk(a, topk: int, jacc_th: float) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    at = transpose_pattern(a)
    out = P(orc_candidate)()
    n = lib().orc_spgemm_topk(a.nrows, _p(arp), _p(aci), _p(at.row_ptr), _p(at.col_idx), topk,
                              jacc_th, C.byref(out))
    res = np.zeros(n, CAND)
    if n:
        raw = C.cast(out, P(C.c_char * (n * CAND.itemsize))).contents
        res = np.frombuffer(bytes(raw), dtype=CAND).copy()
    lib().orc_free(C.cast(out, vp))
    return res


def jaccard(a, i: int, j: int) -> float:
    arp, aci, _ = _csr_args(a)
    return float(lib().orc_jaccard(_p(arp), _p(aci), i, j))


def _cluster_to_dict(c: orc_cluster) -> dict:
    nc, ncs, ns, n = c.nclusters, c.ncolslots, c.nslots, c.nrows
    arr = lambda p, k: np.ctypeslib.as_array(p, shape=(max(k, 1),))[:k].copy()
    d = {"nclusters": nc, "nrows": n, "ncols": c.ncols,
         "cluster_sizes": arr(c.cluster_sizes, nc), "cluster_col_ptr": arr(c.cluster_col_ptr, nc + 1),
         "col_idx": arr(c.col_idx, ncs), "value_ptr": arr(c.value_ptr, nc + 1),
         "values": arr(c.values, ns), "valid": arr(c.valid, (ns + 63) // 64),
         "row_map": arr(c.row_map, n)}
    return d


def build_csr_cluster(a, cluster_ptr: np.ndarray, rows: np.ndarray) -> dict:
    arp, aci, av = _csr_args(a)
    cp = np.ascontiguousarray(cluster_ptr, np.int64)
    rr = np.ascontiguousarray(rows, np.int32)
    c = orc_cluster()
    lib().orc_build_csr_cluster(a.nrows, a.ncols, _p(arp), _p(aci), _p(av), cp.size - 1, _p(cp),
                                _p(rr), C.byref(c))
    d = _cluster_to_dict(c)
    lib().orc_cluster_free(C.byref(c))
    return d


def spgemm_clusterwise(a, cluster_ptr, rows, b):
    """Returns (cluster_to_csr(C) as Csr, C-format dict, access stats tuple)."""
    arp, aci, av = _csr_args(a)
    brp, bci, bv = _csr_args(b)
    cp = np.ascontiguousarray(cluster_ptr, np.int64)
    rr = np.ascontiguousarray(rows, np.int32)
    ac = orc_cluster()
    lib().orc_build_csr_cluster(a.nrows, a.ncols, _p(arp), _p(aci), _p(av), cp.size - 1, _p(cp),
                                _p(rr), C.byref(ac))
    cc = orc_cluster()
    st = orc_access_stats()
    lib().orc_spgemm_clusterwise(C.byref(ac), b.ncols, _p(brp), _p(bci), _p(bv), C.byref(cc),
                                 C.byref(st))
    crp = np.zeros(a.nrows + 1, np.int64)
    ci, cv = P(i32)(), P(dbl)()
    nnz = lib().orc_cluster_to_csr(C.byref(cc), _p(crp), C.byref(ci), C.byref(cv))
    csr = Csr(a.nrows, b.ncols, crp, _arr(ci, nnz, np.int32, lib().orc_free),
              _arr(cv, nnz, np.float64, lib().orc_free))
    d = _cluster_to_dict(cc)
    lib().orc_cluster_free(C.byref(ac))
    lib().orc_cluster_free(C.byref(cc))
    return csr, d, (st.b_row_loads, st.a_inner_iters, st.placeholder_skips)


def merge_candidates(a, pairs: np.ndarray, jacc_th: float, max_cluster: int):
    """Returns (cluster_ptr, rows) of the merge (reference clustering.hpp:122-183)."""
    arp, aci, _ = _csr_args(a)
    pr = np.ascontiguousarray(pairs, CAND)
    cl = np.zeros(a.nrows, np.int32)
    nc = lib().orc_merge_candidates(a.nrows, _p(arp), _p(aci), _p(pr), pr.size, jacc_th,
                                    max_cluster, _p(cl))
    order = np.argsort(cl, kind="stable")
    ptr = np.zeros(nc + 1, np.int64)
    ptr[1:] = np.cumsum(np.bincount(cl, minlength=nc))
    return ptr, order.astype(np.int32)


# ------------------------------------------------------------ reference build
def _ref_check(rc):
    if rc != 0:
        msg = ref().ref_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)


def ref_spgemm_rowwise(a, b, r0: int = 0, r1: int | None = None, threads: int = 0) -> Csr:
    r1 = a.nrows if r1 is None else r1
    arp, aci, av = _csr_args(a)
    brp, bci, bv = _csr_args(b)
    nnz = i64()
    crp, cci, cv = P(i64)(), P(i32)(), P(dbl)()
    _ref_check(ref().ref_spgemm_rowwise(a.nrows, a.ncols, _p(arp), _p(aci), _p(av), b.nrows, b.ncols,
                                        _p(brp), _p(bci), _p(bv), r0, r1, threads, C.byref(nnz),
                                        C.byref(crp), C.byref(cci), C.byref(cv)))
    f = ref().ref_free
    n = nnz.value
    return Csr(r1 - r0, b.ncols, _arr(crp, r1 - r0 + 1, np.int64, f), _arr(cci, n, np.int32, f),
               _arr(cv, n, np.float64, f))


def ref_spgemm_symbolic(a, b, threads: int = 0) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    brp, bci, _ = _csr_args(b)
    out = np.zeros(a.nrows, np.int64)
    _ref_check(ref().ref_spgemm_symbolic(a.nrows, a.ncols, _p(arp), _p(aci), b.nrows, b.ncols,
                                         _p(brp), _p(bci), threads, _p(out)))
    return out


def ref_spgemm_topk(a, topk: int, jacc_th: float, threads: int = 0) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    n = i64()
    out = P(orc_candidate)()
    _ref_check(ref().ref_spgemm_topk(a.nrows, a.ncols, _p(arp), _p(aci), topk, jacc_th, threads,
                                     C.byref(n), C.byref(out)))
    cnt = n.value
    res = np.zeros(cnt, CAND)
    if cnt:
        raw = C.cast(out, P(C.c_char * (cnt * CAND.itemsize))).contents
        res = np.frombuffer(bytes(raw), dtype=CAND).copy()
    ref().ref_free(C.cast(out, vp))
    return res


def _ref_asg(fn, *args):
    nc = i64()
    ptr, rows = P(i64)(), P(i32)()
    _ref_check(fn(*args, C.byref(nc), C.byref(ptr), C.byref(rows)))
    p = _arr(ptr, nc.value + 1, np.int64, ref().ref_free)
    r = _arr(rows, int(p[-1]), np.int32, ref().ref_free)
    return p, r


def ref_hierarchical_clusters(a, jacc_th=0.3, max_cluster=8, threads: int = 0):
    arp, aci, _ = _csr_args(a)
    return _ref_asg(ref().ref_hierarchical_clusters, a.nrows, a.ncols, _p(arp), _p(aci), jacc_th,
                    max_cluster, threads)


def ref_variable_length_clusters(a, jacc_th=0.3, max_cluster=8):
    arp, aci, _ = _csr_args(a)
    return _ref_asg(ref().ref_variable_length_clusters, a.nrows, a.ncols, _p(arp), _p(aci),
                    jacc_th, max_cluster)


def ref_spgemm_clusterwise(a, cluster_ptr, rows, b, threads: int = 0):
    arp, aci, av = _csr_args(a)
    brp, bci, bv = _csr_args(b)
    cp = np.ascontiguousarray(cluster_ptr, np.int64)
    rr = np.ascontiguousarray(rows, np.int32)
    nnz = i64()
    crp, cci, cv = P(i64)(), P(i32)(), P(dbl)()
    st = np.zeros(3, np.uint64)
    slots, colslots = i64(), i64()
    _ref_check(ref().ref_spgemm_clusterwise(a.nrows, a.ncols, _p(arp), _p(aci), _p(av), b.nrows,
                                            b.ncols, _p(brp), _p(bci), _p(bv), cp.size - 1, _p(cp),
                                            _p(rr), threads, C.byref(nnz), C.byref(crp),
                                            C.byref(cci), C.byref(cv), _p(st), C.byref(slots),
                                            C.byref(colslots)))
    f = ref().ref_free
    n = nnz.value
    csr = Csr(a.nrows, b.ncols, _arr(crp, a.nrows + 1, np.int64, f), _arr(cci, n, np.int32, f),
              _arr(cv, n, np.float64, f))
    return csr, tuple(int(x) for x in st), int(slots.value), int(colslots.value)


def ref_reorder_rcm(a) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    out = np.zeros(a.nrows, np.int32)
    _ref_check(ref().ref_reorder_rcm(a.nrows, a.ncols, _p(arp), _p(aci), _p(out)))
    return out


def ref_reorder_random(n: int, seed: int) -> np.ndarray:
    out = np.zeros(n, np.int32)
    _ref_check(ref().ref_reorder_random(n, seed, _p(out)))
    return out


def ref_reorder_degree(a) -> np.ndarray:
    arp, aci, _ = _csr_args(a)
    out = np.zeros(a.nrows, np.int32)
    _ref_check(ref().ref_reorder_degree(a.nrows, a.ncols, _p(arp), _p(aci), _p(out)))
    return out


def ref_permute_symmetric(a, perm) -> Csr:
    arp, aci, av = _csr_args(a)
    pp = np.ascontiguousarray(perm, np.int32)
    rp, ci, v = P(i64)(), P(i32)(), P(dbl)()
    _ref_check(ref().ref_permute_symmetric(a.nrows, a.ncols, _p(arp), _p(aci), _p(av), _p(pp),
                                           C.byref(rp), C.byref(ci), C.byref(v)))
    f = ref().ref_free
    rpa = _arr(rp, a.nrows + 1, np.int64, f)
    nnz = int(rpa[-1])
    return Csr(a.nrows, a.ncols, rpa, _arr(ci, nnz, np.int32, f), _arr(v, nnz, np.float64, f))


def ref_jaccard(a, i, j) -> float:
    arp, aci, _ = _csr_args(a)
    out = dbl()
    _ref_check(ref().ref_jaccard(a.nrows, a.ncols, _p(arp), _p(aci), i, j, C.byref(out)))
    return float(out.value)


def ref_generate_frontiers(a, num_frontiers: int, batch: int, seed: int) -> list:
    """The reference's generate_frontiers (frontier.hpp:20-77) on host CSR `a`."""
    arp, aci, _ = _csr_args(a)
    cnt, width = i64(), i64()
    rps, coff, cis = P(i64)(), P(i64)(), P(i32)()
    _ref_check(ref().ref_generate_frontiers(a.nrows, a.ncols, _p(arp), _p(aci), num_frontiers,
                                            batch, seed, C.byref(cnt), C.byref(width),
                                            C.byref(rps), C.byref(coff), C.byref(cis)))
    f = ref().ref_free
    n, k = a.nrows, cnt.value
    rp = _arr(rps, k * (n + 1), np.int64, f).reshape(k, n + 1) if k else np.zeros((0, n + 1), np.int64)
    off = _arr(coff, k + 1, np.int64, f)
    ci = _arr(cis, int(off[-1]), np.int32, f)
    return [Csr(n, width.value, rp[t].copy(), ci[off[t]:off[t + 1]].copy(),
                np.ones(off[t + 1] - off[t], np.float64)) for t in range(k)]


# ---------------------------------------------------------------------------
# Frontier generation (restatement of frontier.hpp:20-77, pure Python: small
# inputs only).  std::mt19937_64 per the C++ standard [rand.eng.mers] and the
# reference's multiply-shift `bounded` (types.hpp:36-39).
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


class _MT19937_64:
    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _M64
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _M64
        self.i = 312

    def __call__(self) -> int:
        if self.i >= 312:
            mt = self.mt
            for k in range(312):
                x = (mt[k] & 0xFFFFFFFF80000000) | (mt[(k + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                mt[k] = mt[(k + 156) % 312] ^ xa
            self.i = 0
        x = self.mt[self.i]
        self.i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        return x & _M64


def random_permutation(n: int, seed: int) -> np.ndarray:
    """reorder_random (reorder.hpp:20-30): Fisher-Yates, j = (rng() * (i+1)) >> 64."""
    rng = _MT19937_64(seed)
    perm = list(range(n))
    for i in range(n - 1, 0, -1):
        j = (rng() * (i + 1)) >> 64
        perm[i], perm[j] = perm[j], perm[i]
    return np.array(perm, np.int32)


def generate_frontiers(a, num_frontiers: int, batch: int, seed: int) -> list:
    """frontier.hpp:20-77: `width = min(batch, n)` sorted sources from the first
    entries of a seeded shuffle (:37-46); one BFS per source over a's rows as
    out-neighbour lists (:48-63); frontier t = {(v, s): depth_s(v) == t}
    (:65-76), at most num_frontiers of them, fewer when every search ends."""
    if a.nrows != a.ncols or num_frontiers < 1 or batch < 1:
        raise ValueError("generate_frontiers: contract")
    n = a.nrows
    if n == 0:
        return []
    width = min(batch, n)
    sources = np.sort(random_permutation(n, seed)[:width])
    rp, ci = np.asarray(a.row_ptr, np.int64), np.asarray(a.col_idx, np.int32)
    depth = np.full((width, n), -1, np.int64)
    max_depth = 0
    for s in range(width):
        d = depth[s]
        q = [int(sources[s])]
        d[q[0]] = 0
        h = 0
        while h < len(q):
            v = q[h]
            h += 1
            for w in ci[rp[v]:rp[v + 1]]:
                if d[w] < 0:
                    d[w] = d[v] + 1
                    q.append(int(w))
        max_depth = max(max_depth, int(d[q[-1]]))
    out = []
    for t in range(min(num_frontiers, max_depth + 1)):
        vv, ss = np.nonzero(depth.T == t)  # row-major over (v, s): rows sorted, cols ascending
        cnt = np.bincount(vv, minlength=n)
        rpt = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
        out.append(Csr(n, width, rpt, ss.astype(np.int32), np.ones(len(ss), np.float64)))
    return out


# ------------------------------------------------------------ generator (gen.c)
def gen_rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int) -> Csr:
    """The cfg3/cfg5 R-MAT recipe restated in C (gen.c), bit-identical to the
    product's generator (tests/test_oracle.py) — bench.py's reference arm builds its
    input with it, so that process never loads the product library."""
    n = i64()
    rp, ci, v = P(i64)(), P(i32)(), P(dbl)()
    rc = lib().orc_gen_rmat(scale, edge_factor, a, b, c, seed, C.byref(n), C.byref(rp),
                            C.byref(ci), C.byref(v))
    if rc != 0:
        raise ValueError("orc_gen_rmat: bad sizes or out of memory")
    f = lib().orc_free
    nn = n.value
    row_ptr = _arr(rp, nn + 1, np.int64, f)
    nnz = int(row_ptr[-1])
    return Csr(nn, nn, row_ptr, _arr(ci, nnz, np.int32, f), _arr(v, nnz, np.float64, f))


# ------------------------------------------------ reference timing (bench only)
class RefCsr:
    """The reference's own CsrMatrix (int32 offsets), built once outside any timed
    region (ref_shim.cpp ref_csr_new)."""

    def __init__(self, a):
        arp, aci, av = _csr_args(a)
        self.nrows, self.ncols = a.nrows, a.ncols
        self.h = ref().ref_csr_new(a.nrows, a.ncols, _p(arp), _p(aci), _p(av))
        if not self.h:
            _ref_check(6)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_csr_delete(self.h)
            self.h = None


class RefCluster:
    """The reference's CsrClusterMatrix of a RefCsr and an assignment
    (build_csr_cluster, cluster_format.hpp:130-186), built outside the timing."""

    def __init__(self, a: RefCsr, cluster_ptr, rows):
        cp = np.ascontiguousarray(cluster_ptr, np.int64)
        rr = np.ascontiguousarray(rows, np.int32)
        self.h = ref().ref_cluster_new(a.h, cp.size - 1, _p(cp), _p(rr))
        if not self.h:
            _ref_check(6)

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_cluster_delete(self.h)
            self.h = None


def ref_time_rowwise(a: RefCsr, b: RefCsr, threads: int = 0):
    """Seconds of the reference's spgemm_rowwise(a, b) call alone (and nnz(C))."""
    s, nnz = dbl(), i64()
    _ref_check(ref().ref_time_rowwise(a.h, b.h, threads, C.byref(s), C.byref(nnz)))
    return s.value, nnz.value


def ref_time_clusterwise(ac: RefCluster, b: RefCsr, threads: int = 0):
    """Seconds of the reference's spgemm_clusterwise(ac, b) call alone (and C's
    value slots)."""
    s, slots = dbl(), i64()
    _ref_check(ref().ref_time_clusterwise_prepared(ac.h, b.h, threads, C.byref(s),
                                                   C.byref(slots)))
    return s.value, slots.value


def ref_load_matrix_market(path) -> Csr:
    """The reference's load_matrix_market + coo_to_csr (matrix_market.hpp:42-119)."""
    nr, nc, nz = i64(), i64(), i64()
    crp, cci, cv = P(i64)(), P(i32)(), P(dbl)()
    _ref_check(ref().ref_load_matrix_market(str(path).encode(), C.byref(nr), C.byref(nc),
                                            C.byref(nz), C.byref(crp), C.byref(cci), C.byref(cv)))
    f = ref().ref_free
    return Csr(nr.value, nc.value, _arr(crp, nr.value + 1, np.int64, f),
               _arr(cci, nz.value, np.int32, f), _arr(cv, nz.value, np.float64, f))


def ref_load_permutation(path, nrows: int) -> np.ndarray:
    out = np.zeros(nrows, np.int32)
    _ref_check(ref().ref_load_permutation(str(path).encode(), nrows, _p(out)))
    return out


def ref_write_matrix_market(a, path) -> None:
    arp, aci, av = _csr_args(a)
    _ref_check(ref().ref_write_matrix_market(a.nrows, a.ncols, _p(arp), _p(aci), _p(av),
                                             str(path).encode()))


def ref_fmt_double(v: float) -> str:
    """std::to_chars(double) as the reference's CSV writer uses it."""
    buf = C.create_string_buffer(64)
    _ref_check(ref().ref_fmt_double(v, buf, 64))
    return buf.value.decode()


def ref_bench_csv_row(matrix, workload, reorder_method, reorder_seed, reorder_path,
                      cluster_method, jacc_th, max_cluster, fixed_len, nf, fb, fseed, reps,
                      threads, warmup, d9, u6, ratio, amort):
    """(row, header) as the reference's bench_csv_row / bench_csv_header print them."""
    d = np.ascontiguousarray(d9, np.float64)
    u = np.ascontiguousarray(u6, np.uint64)
    buf = C.create_string_buffer(1 << 12)
    _ref_check(ref().ref_bench_csv_row(str(matrix).encode(), workload, reorder_method, reorder_seed,
                                       str(reorder_path).encode(), cluster_method, jacc_th,
                                       max_cluster, fixed_len, nf, fb, fseed, reps, threads,
                                       warmup, _p(d), _p(u), ratio, amort, buf, 1 << 12))
    row, header = buf.value.decode().split("\n")
    return row, header
