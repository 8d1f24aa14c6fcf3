"""B200-native cluster-wise SpGEMM engine (host-side Python mirror of the
reference's ``namespace cspgemm`` API, over the C ABI in include/bsp.h).

Reference interface mirrored (paths under /root/reference/proj/include/cspgemm):
  CsrMatrix (csr.hpp:51-88), Permutation (permutation.hpp), ClusterAssignment
  (cluster_format.hpp:23-59), CsrClusterMatrix (:94-125), spgemm_symbolic /
  spgemm_rowwise / jaccard_similarity / spgemm_topk (spgemm.hpp:41-206),
  build_csr_cluster / cluster_to_csr (cluster_format.hpp:130-233),
  spgemm_clusterwise[_instrumented] (cluster_spgemm.hpp:186-197),
  fixed/variable/hierarchical clustering (clustering.hpp:59-194),
  reorder_random / reorder_degree / reorder_rcm / bandwidth (reorder.hpp),
  transpose / binarize / permute_symmetric / permute_rows (csr.hpp:115-193).

Every multiply runs on the GPU through libbsp.so; there is no CPU fallback.
Errors mirror the reference: ``ContractError`` (a ``ValueError``, like
``std::invalid_argument``) for precondition violations.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Tuple, Iterable, List, Optional, Sequence

import numpy as np

from . import _lib as L

__all__ = [
    "ContractError", "BspError", "CsrMatrix", "Permutation", "ClusterAssignment", "ClusterParams",
    "CandidatePair", "AccessStats", "Engine", "DeviceCsr", "DeviceCsrCluster", "default_engine",
    "spgemm_symbolic", "spgemm_rowwise", "spgemm_topk", "jaccard_similarity",
    "build_csr_cluster", "cluster_to_csr", "spgemm_clusterwise", "spgemm_clusterwise_instrumented",
    "rowwise_access_stats", "fixed_length_clusters", "variable_length_clusters",
    "hierarchical_clusters", "merge_candidates", "assignment_to_permutation", "reorder_random",
    "reorder_degree", "reorder_rcm", "bandwidth", "transpose", "generate_frontiers", "binarize",
    "permute_symmetric",
    "permute_rows", "coo_to_csr", "csr_equal_canonical", "gen_er", "gen_hidden_clusters",
    "gen_rmat", "gen_stencil27", "make_config", "CONFIGS", "load_matrix_market",
    "write_matrix_market", "load_permutation", "write_permutation", "ReorderSpec",
    "make_permutation",
]


class BspError(RuntimeError):
    """Device/engine failure (CUDA error, out of memory, internal)."""


class ContractError(ValueError):
    """Precondition violation; mirrors cspgemm::contract_error (types.hpp:16-19)."""


class BspIOError(RuntimeError):
    """Mirrors cspgemm::io_error (types.hpp:23-26)."""


def _check(rc: int) -> None:
    if rc == L.BSP_OK:
        return
    msg = L.load().bsp_last_error().decode(errors="replace")
    if rc == L.BSP_ERR_CONTRACT:
        raise ContractError(msg)
    if rc == L.BSP_ERR_IO:
        raise BspIOError(msg)
    if rc == L.BSP_ERR_OOM:
        raise MemoryError(msg)
    raise BspError(msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


# ---------------------------------------------------------------------------
# host types
# ---------------------------------------------------------------------------
@dataclass
class CsrMatrix:
    """Host CSR (reference csr.hpp:51-88) with int64 row offsets."""

    nrows: int
    ncols: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int32)
        self.values = np.ascontiguousarray(self.values, dtype=np.float64)
        self.nrows = int(self.nrows)
        self.ncols = int(self.ncols)

    def nnz(self) -> int:
        return int(self.row_ptr[self.nrows]) if self.row_ptr.size else 0

    def row_nnz(self, i: int) -> int:
        return int(self.row_ptr[i + 1] - self.row_ptr[i])

    def row_cols(self, i: int) -> np.ndarray:
        return self.col_idx[self.row_ptr[i]:self.row_ptr[i + 1]]

    def row_vals(self, i: int) -> np.ndarray:
        return self.values[self.row_ptr[i]:self.row_ptr[i + 1]]

    def check_invariants(self) -> None:
        """reference csr.hpp:70-87."""
        rp, ci = self.row_ptr, self.col_idx
        if rp.size != self.nrows + 1:
            raise ContractError("csr: row_ptr length must be nrows+1")
        if rp[0] != 0:
            raise ContractError("csr: row_ptr[0] must be 0")
        if np.any(np.diff(rp) < 0):
            raise ContractError("csr: row_ptr must be non-decreasing")
        if ci.size and (ci.min() < 0 or ci.max() >= self.ncols):
            raise ContractError("csr: column index out of range")
        if rp[-1] != ci.size:
            raise ContractError("csr: row_ptr[nrows] must equal nnz")
        if ci.size != self.values.size:
            raise ContractError("csr: col_idx/values length mismatch")
        if ci.size > 1:
            d = np.diff(ci.astype(np.int64))
            starts = np.zeros(ci.size - 1, dtype=bool)
            inner = rp[1:-1]
            inner = inner[(inner > 0) & (inner < ci.size)]
            starts[inner - 1] = True
            if np.any((d <= 0) & ~starts):
                raise ContractError("csr: columns must be strictly increasing within a row")

    def _host(self) -> L.bsp_host_csr:
        s = L.bsp_host_csr()
        s.nrows, s.ncols, s.nnz = self.nrows, self.ncols, self.nnz()
        s.row_ptr = self.row_ptr.ctypes.data_as(C.POINTER(C.c_int64))
        s.col_idx = self.col_idx.ctypes.data_as(C.POINTER(C.c_int32))
        s.values = self.values.ctypes.data_as(C.POINTER(C.c_double))
        return s

    @staticmethod
    def _adopt(s: L.bsp_host_csr) -> "CsrMatrix":
        """Copy a library-malloc'ed host CSR into numpy and free it."""
        n, nnz = int(s.nrows), int(s.nnz)
        rp = np.ctypeslib.as_array(s.row_ptr, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(s.col_idx, shape=(nnz,)).copy() if nnz else np.zeros(0, np.int32)
        v = np.ctypeslib.as_array(s.values, shape=(nnz,)).copy() if nnz else np.zeros(0)
        L.load().bsp_host_csr_free(C.byref(s))
        return CsrMatrix(n, int(s.ncols), rp, ci, v)

    def copy(self) -> "CsrMatrix":
        return CsrMatrix(self.nrows, self.ncols, self.row_ptr.copy(), self.col_idx.copy(),
                         self.values.copy())

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.nrows, self.ncols))
        rows = np.repeat(np.arange(self.nrows), np.diff(self.row_ptr))
        np.add.at(d, (rows, self.col_idx), self.values)
        return d


def coo_to_csr(nrows: int, ncols: int, rows, cols, vals) -> CsrMatrix:
    """reference csr.hpp:92-113: sort by (row, col), sum duplicates."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    if rows.size and (rows.min() < 0 or rows.max() >= nrows):
        raise ContractError("coo_to_csr: row index out of range")
    if cols.size and (cols.min() < 0 or cols.max() >= ncols):
        raise ContractError("coo_to_csr: col index out of range")
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        key = rows * max(ncols, 1) + cols
        first = np.ones(rows.size, dtype=bool)
        first[1:] = key[1:] != key[:-1]
        idx = np.flatnonzero(first)
        summed = np.add.reduceat(vals, idx) if idx.size else vals
        rows, cols, vals = rows[idx], cols[idx], summed
    rp = np.zeros(nrows + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return CsrMatrix(nrows, ncols, np.cumsum(rp), cols.astype(np.int32), vals)


def binarize(a: CsrMatrix) -> CsrMatrix:
    """reference csr.hpp:138-142."""
    return CsrMatrix(a.nrows, a.ncols, a.row_ptr.copy(), a.col_idx.copy(), np.ones(a.nnz()))


def csr_equal_canonical(a: CsrMatrix, b: CsrMatrix, tol: float) -> bool:
    """reference csr.hpp:197-203."""
    if a.nrows != b.nrows or a.ncols != b.ncols:
        return False
    if not np.array_equal(a.row_ptr, b.row_ptr) or not np.array_equal(a.col_idx, b.col_idx):
        return False
    return bool(np.all(np.abs(a.values - b.values) <= tol))


@dataclass
class Permutation:
    """reference permutation.hpp: perm[new] = old, inv[old] = new."""

    perm: np.ndarray
    inv: np.ndarray = None

    def __post_init__(self):
        self.perm = np.ascontiguousarray(self.perm, dtype=np.int32)
        if self.inv is None:
            n = self.perm.size
            if n and (self.perm.min() < 0 or self.perm.max() >= n):
                bad = int(self.perm[(self.perm < 0) | (self.perm >= n)][0])
                raise ContractError(f"permutation: index {bad} out of range")
            inv = np.full(n, -1, dtype=np.int32)
            inv[self.perm] = np.arange(n, dtype=np.int32)
            if n and np.any(inv < 0):
                vals, counts = np.unique(self.perm, return_counts=True)
                raise ContractError(f"permutation: duplicate index {int(vals[counts > 1][0])}")
            self.inv = inv

    @property
    def size(self) -> int:
        return int(self.perm.size)

    @staticmethod
    def identity(n: int) -> "Permutation":
        return Permutation(np.arange(n, dtype=np.int32))

    @staticmethod
    def from_perm(p: Sequence[int]) -> "Permutation":
        return Permutation(np.asarray(p, dtype=np.int32))

    def inverse(self) -> "Permutation":
        return Permutation(self.inv.copy(), self.perm.copy())


class ClusterAssignment:
    """reference cluster_format.hpp:23-59, stored flattened (cluster_ptr, rows)."""

    def __init__(self, cluster_ptr: np.ndarray, rows: np.ndarray):
        self.cluster_ptr = np.ascontiguousarray(cluster_ptr, dtype=np.int64)
        self.rows = np.ascontiguousarray(rows, dtype=np.int32)

    @staticmethod
    def from_lists(clusters: Iterable[Sequence[int]]) -> "ClusterAssignment":
        cl = [list(c) for c in clusters]
        ptr = np.zeros(len(cl) + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([len(c) for c in cl]) if cl else []
        rows = np.array([r for c in cl for r in c], dtype=np.int32)
        return ClusterAssignment(ptr, rows)

    @staticmethod
    def singletons(n: int) -> "ClusterAssignment":
        return ClusterAssignment(np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32))

    @property
    def nclusters(self) -> int:
        return int(self.cluster_ptr.size - 1)

    def nrows(self) -> int:
        return int(self.rows.size)

    @property
    def clusters(self) -> List[List[int]]:
        return [self.rows[self.cluster_ptr[c]:self.cluster_ptr[c + 1]].tolist()
                for c in range(self.nclusters)]

    def sizes(self) -> np.ndarray:
        return np.diff(self.cluster_ptr)

    def validate(self, nrows: int) -> None:
        """reference cluster_format.hpp:34-51."""
        seen = np.zeros(nrows, dtype=bool)
        for c in range(self.nclusters):
            m = self.rows[self.cluster_ptr[c]:self.cluster_ptr[c + 1]]
            if m.size == 0:
                raise ContractError("cluster assignment: empty cluster")
            if m.min() < 0 or m.max() >= nrows:
                raise ContractError("cluster assignment: row index out of range")
            if np.any(seen[m]):
                raise ContractError("cluster assignment: row assigned twice")
            seen[m] = True
            if np.any(np.diff(m) <= 0):
                raise ContractError("cluster assignment: members must be strictly increasing")
        if not seen.all():
            raise ContractError(f"cluster assignment: row {int(np.argmin(seen))} not covered")

    def __eq__(self, other) -> bool:
        return (isinstance(other, ClusterAssignment)
                and np.array_equal(self.cluster_ptr, other.cluster_ptr)
                and np.array_equal(self.rows, other.rows))

    @staticmethod
    def _adopt(nc: int, ptr, rows) -> "ClusterAssignment":
        lib = L.load()
        p = np.ctypeslib.as_array(ptr, shape=(nc + 1,)).copy()
        total = int(p[-1])
        r = np.ctypeslib.as_array(rows, shape=(total,)).copy() if total else np.zeros(0, np.int32)
        lib.bsp_host_free_plain(C.cast(ptr, C.c_void_p))
        lib.bsp_host_free_plain(C.cast(rows, C.c_void_p))
        return ClusterAssignment(p, r)


@dataclass
class ClusterParams:
    """reference clustering.hpp:52-56 (defaults jacc 0.3, max 8, fixed 4)."""

    jacc_th: float = 0.3
    max_cluster_th: int = 8
    fixed_len: int = 4


CandidatePair = np.dtype([("i", np.int32), ("j", np.int32), ("score", np.float64)])


@dataclass
class AccessStats:
    """reference cluster_spgemm.hpp:26-30."""

    b_row_loads: int = 0
    a_inner_iters: int = 0
    placeholder_skips: int = 0


# ---------------------------------------------------------------------------
# device objects
# ---------------------------------------------------------------------------
class DeviceCsr:
    """A device-resident CSR (bsp_csr) owned by an Engine."""

    def __init__(self, engine: "Engine", s: L.bsp_csr, keep=None):
        self.engine = engine
        self.s = s
        self._keep = keep  # keeps viewed buffers (e.g. torch tensors) alive

    nrows = property(lambda self: int(self.s.nrows))
    ncols = property(lambda self: int(self.s.ncols))

    def nnz(self) -> int:
        return int(self.s.nnz)

    def torch_views(self):
        """Zero-copy torch views (row_ptr int64, col_idx int32, values float64) of
        this device CSR's arrays (valid while it lives)."""
        import torch

        class _Cai:
            def __init__(s_, ptr, n, ts):
                s_.__cuda_array_interface__ = {"shape": (n,), "typestr": ts,
                                               "data": (int(ptr or 0), False), "version": 3}

        dev = f"cuda:{self.engine.device}"
        return (torch.as_tensor(_Cai(self.s.row_ptr, self.nrows + 1, "<i8"), device=dev),
                torch.as_tensor(_Cai(self.s.col_idx, self.nnz(), "<i4"), device=dev),
                torch.as_tensor(_Cai(self.s.values, self.nnz(), "<f8"), device=dev))

    def download(self) -> CsrMatrix:
        n, nnz = self.nrows, self.nnz()
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.int32)
        v = np.empty(nnz, np.float64)
        _check(self.engine.lib.bsp_csr_download(self.engine.h, C.byref(self.s), _ptr(rp), _ptr(ci),
                                                _ptr(v)))
        return CsrMatrix(n, self.ncols, rp, ci, v)

    def download_async(self, row_ptr: int, col_idx: int, values: int,
                       engine: Optional["Engine"] = None) -> None:
        """Enqueue D2H copies into caller buffers (e.g. pinned) on `engine`'s stream."""
        e = engine or self.engine
        _check(e.lib.bsp_csr_download_async(e.h, C.byref(self.s), row_ptr, col_idx, values))

    def free(self, engine: Optional["Engine"] = None) -> None:
        """Release (stream-ordered on `engine`'s stream, default the owner's)."""
        e = engine or self.engine
        if self.s is not None and e.h:
            e.lib.bsp_csr_free(e.h, C.byref(self.s))
        self.s = None

    def __del__(self):
        try:
            if self.s is not None and self.s.owned:
                self.free()
        except Exception:
            pass


class DeviceCsrCluster:
    """Device CSR_Cluster (bsp_csr_cluster)."""

    def __init__(self, engine: "Engine", s: L.bsp_csr_cluster):
        self.engine = engine
        self.s = s

    nclusters = property(lambda self: int(self.s.nclusters))
    nrows = property(lambda self: int(self.s.nrows))
    ncols = property(lambda self: int(self.s.ncols))

    def value_slots(self) -> int:
        return int(self.s.nslots)

    def download(self) -> dict:
        h = L.bsp_host_csr_cluster()
        lib = self.engine.lib
        _check(lib.bsp_csr_cluster_download(self.engine.h, C.byref(self.s), C.byref(h)))
        nc, ncs, ns, n = int(h.nclusters), int(h.ncolslots), int(h.nslots), int(h.nrows)
        arr = np.ctypeslib.as_array
        out = {
            "nclusters": nc, "nrows": n, "ncols": int(h.ncols),
            "cluster_sizes": arr(h.cluster_sizes, (max(nc, 1),))[:nc].copy(),
            "cluster_col_ptr": arr(h.cluster_col_ptr, (nc + 1,)).copy(),
            "col_idx": arr(h.col_idx, (max(ncs, 1),))[:ncs].copy(),
            "value_ptr": arr(h.value_ptr, (nc + 1,)).copy(),
            "values": arr(h.values, (max(ns, 1),))[:ns].copy(),
            "valid": arr(h.valid, (max((ns + 63) // 64, 1),))[:(ns + 63) // 64].copy(),
            "row_map": arr(h.row_map, (max(n, 1),))[:n].copy(),
        }
        lib.bsp_host_csr_cluster_free(C.byref(h))
        out["placeholders"] = ns - int(sum(bin(int(w)).count("1") for w in out["valid"]))
        return out

    def free(self) -> None:
        # after Engine.close() the handle (its stream and pools) is gone: drop
        if self.s is not None and self.engine.h:
            self.engine.lib.bsp_csr_cluster_free(self.engine.h, C.byref(self.s))
        self.s = None

    def __del__(self):
        try:
            if self.s is not None and self.s.owned:
                self.free()
        except Exception:
            pass


class Engine:
    """One bsp handle (device, stream, memory pool)."""

    def __init__(self, device: int = 0):
        self.lib = L.load()
        h = C.c_void_p()
        _check(self.lib.bsp_create(device, C.byref(h)))
        self.h = h
        self.device = device

    def close(self) -> None:
        if self.h:
            self.lib.bsp_destroy(self.h)
            self.h = None

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        _check(self.lib.bsp_set_stream(self.h, stream_ptr))

    def stream_ptr(self) -> int:
        return int(self.lib.bsp_get_stream(self.h) or 0)

    def wait_for(self, other: "Engine") -> None:
        """This engine's stream waits for the work enqueued on `other`'s."""
        _check(self.lib.bsp_stream_wait(self.h, other.h))

    def synchronize(self) -> None:
        _check(self.lib.bsp_synchronize(self.h))

    def profile(self, on: bool = True) -> None:
        _check(self.lib.bsp_profile(self.h, 1 if on else 0))

    def profile_report(self) -> dict:
        """{kernel name: (launches, total ms)} since the last report."""
        buf = C.create_string_buffer(1 << 16)
        n = self.lib.bsp_profile_report(self.h, buf, 1 << 16)
        if n < 0:
            raise BspError(self.lib.bsp_last_error().decode())
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ms = line.split("\t")
            out[name] = (int(cnt), float(ms))
        return out

    def kernel_launches(self) -> int:
        return int(self.lib.bsp_kernel_launches(self.h))

    def exec_stats(self) -> dict:
        s = L.bsp_exec_stats()
        _check(self.lib.bsp_get_exec_stats(self.h, C.byref(s)))
        return {"products": s.products, "nnz_out": s.nnz_out, "units": list(s.units),
                "kernels_launched": s.kernels_launched, "chunks": s.chunks}

    # -- transfers ---------------------------------------------------------
    def upload(self, a: CsrMatrix) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_csr_upload(self.h, a.nrows, a.ncols, _ptr(a.row_ptr), _ptr(a.col_idx),
                                       _ptr(a.values), C.byref(s)))
        return DeviceCsr(self, s)

    def view(self, nrows: int, ncols: int, nnz: int, row_ptr: int, col_idx: int, values: int,
             keep=None) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_csr_view(nrows, ncols, nnz, row_ptr, col_idx, values, C.byref(s)))
        return DeviceCsr(self, s, keep)

    def view_torch(self, nrows: int, ncols: int, row_ptr, col_idx, values) -> DeviceCsr:
        """Zero-copy view of torch CUDA tensors (int64, int32, float64)."""
        return self.view(nrows, ncols, int(col_idx.numel()), row_ptr.data_ptr(),
                         col_idx.data_ptr(), values.data_ptr(), keep=(row_ptr, col_idx, values))

    # -- row-wise ----------------------------------------------------------
    def spgemm_rowwise(self, A: DeviceCsr, B: DeviceCsr) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_spgemm_rowwise(self.h, C.byref(A.s), C.byref(B.s), C.byref(s)))
        return DeviceCsr(self, s)

    def spgemm_rowwise_range(self, A: DeviceCsr, B: DeviceCsr, r0: int, r1: int) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_spgemm_rowwise_range(self.h, C.byref(A.s), C.byref(B.s), r0, r1,
                                                 C.byref(s)))
        return DeviceCsr(self, s)

    def spgemm_symbolic(self, A: DeviceCsr, B: DeviceCsr) -> np.ndarray:
        import torch  # device buffer for the counts

        cnt = torch.empty(max(A.nrows, 1), dtype=torch.int64, device=f"cuda:{self.device}")
        _check(self.lib.bsp_spgemm_symbolic(self.h, C.byref(A.s), C.byref(B.s), cnt.data_ptr()))
        return cnt[:A.nrows].cpu().numpy()

    def spgemm_products(self, A: DeviceCsr, B: DeviceCsr) -> int:
        tot = C.c_int64()
        _check(self.lib.bsp_spgemm_products(self.h, C.byref(A.s), C.byref(B.s), None,
                                            C.byref(tot)))
        return int(tot.value)

    def partition_rows(self, A: DeviceCsr, B: DeviceCsr, nparts: int) -> np.ndarray:
        b = np.zeros(nparts + 1, np.int64)
        _check(self.lib.bsp_partition_rows(self.h, C.byref(A.s), C.byref(B.s), nparts, _ptr(b)))
        return b

    # -- multi-GPU (one process per GPU, NCCL; include/bsp.h "multi-GPU") ----
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(L.BSP_NCCL_ID_BYTES)
        _check(L.load().bsp_nccl_unique_id(buf))
        return buf.raw

    def comm_init(self, nranks: int, rank: int, uid: bytes) -> None:
        """Give this engine its own NCCL communicator (rank of nranks)."""
        buf = C.create_string_buffer(bytes(uid), L.BSP_NCCL_ID_BYTES)
        _check(self.lib.bsp_comm_init(self.h, nranks, rank, buf))

    def comm_destroy(self) -> None:
        _check(self.lib.bsp_comm_destroy(self.h))

    def comm_rank(self) -> Tuple[int, int]:
        r, n = C.c_int(), C.c_int()
        _check(self.lib.bsp_comm_rank(self.h, C.byref(r), C.byref(n)))
        return r.value, n.value

    def broadcast(self, M: Optional[DeviceCsr], root: int = 0) -> Tuple[DeviceCsr, float]:
        """Replicate a device CSR from `root` (NCCL); returns (matrix, ms)."""
        s = M.s if M is not None else L.bsp_csr()
        ms = C.c_double()
        _check(self.lib.bsp_csr_broadcast(self.h, C.byref(s), root, C.byref(ms)))
        return (M if M is not None else DeviceCsr(self, s)), float(ms.value)

    def allgather_rows(self, shard: DeviceCsr) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_csr_allgather_rows(self.h, C.byref(shard.s), C.byref(s)))
        return DeviceCsr(self, s)

    def spgemm_rowwise_sharded(self, A: DeviceCsr, B: DeviceCsr, gather: bool = False):
        """Row-sharded C = A*B over the engine's communicator: (C, info) with C this
        rank's row block, or the global C on every rank when gather=True."""
        s = L.bsp_csr()
        inf = L.bsp_shard_info()
        _check(self.lib.bsp_spgemm_rowwise_sharded(self.h, C.byref(A.s), C.byref(B.s),
                                                   1 if gather else 0, C.byref(s), C.byref(inf)))
        info = {k: getattr(inf, k) for k, _ in L.bsp_shard_info._fields_}
        return DeviceCsr(self, s), info

    def partition_clusters(self, Ac: "DeviceCsrCluster", B: DeviceCsr, nparts: int) -> np.ndarray:
        b = np.zeros(nparts + 1, np.int64)
        _check(self.lib.bsp_partition_clusters(self.h, C.byref(Ac.s), C.byref(B.s), nparts,
                                               _ptr(b)))
        return b

    def select_rows(self, A: DeviceCsr, rows: np.ndarray) -> DeviceCsr:
        import torch

        r = torch.from_numpy(np.ascontiguousarray(rows, np.int32)).to(f"cuda:{self.device}")
        torch.cuda.synchronize(self.device)
        s = L.bsp_csr()
        _check(self.lib.bsp_csr_select_rows(self.h, C.byref(A.s), r.data_ptr(), int(r.numel()),
                                            C.byref(s)))
        self.synchronize()
        return DeviceCsr(self, s)

    def spgemm_rowwise_host(self, a: CsrMatrix, b: CsrMatrix) -> CsrMatrix:
        ha, hb = a._host(), b._host()
        hc = L.bsp_host_csr()
        _check(self.lib.bsp_spgemm_rowwise_host(self.h, C.byref(ha),
                                                C.byref(ha) if b is a else C.byref(hb),
                                                C.byref(hc)))
        return CsrMatrix._adopt(hc)

    def transpose(self, A: DeviceCsr) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_transpose(self.h, C.byref(A.s), C.byref(s)))
        return DeviceCsr(self, s)

    def generate_frontiers(self, A: DeviceCsr, num_frontiers: int = 10, batch: int = 64,
                           seed: int = 0) -> list:
        """Frontier operands of the tall-skinny workload (frontier.hpp:20-77) as
        device CSRs, built by a batched BFS on the device."""
        arr = (L.bsp_csr * max(int(num_frontiers), 1))()
        cnt = C.c_int64()
        _check(self.lib.bsp_generate_frontiers(self.h, C.byref(A.s), num_frontiers, batch, seed,
                                               arr, C.byref(cnt)))
        return [DeviceCsr(self, arr[t]) for t in range(cnt.value)]

    # -- cluster-wise --------------------------------------------------------
    def build_csr_cluster(self, A: DeviceCsr, asg: ClusterAssignment) -> DeviceCsrCluster:
        s = L.bsp_csr_cluster()
        _check(self.lib.bsp_csr_cluster_build(self.h, C.byref(A.s), asg.nclusters,
                                              _ptr(asg.cluster_ptr), _ptr(asg.rows), C.byref(s)))
        return DeviceCsrCluster(self, s)

    def spgemm_clusterwise(self, Ac: DeviceCsrCluster, B: DeviceCsr, want_cluster: bool = False):
        s = L.bsp_csr()
        cs = L.bsp_csr_cluster() if want_cluster else None
        _check(self.lib.bsp_spgemm_clusterwise(self.h, C.byref(Ac.s), C.byref(B.s), C.byref(s),
                                               C.byref(cs) if cs is not None else None))
        out = DeviceCsr(self, s)
        return (out, DeviceCsrCluster(self, cs)) if want_cluster else out

    def cluster_to_csr(self, Ac: DeviceCsrCluster) -> DeviceCsr:
        s = L.bsp_csr()
        _check(self.lib.bsp_cluster_to_csr(self.h, C.byref(Ac.s), C.byref(s)))
        return DeviceCsr(self, s)

    def cluster_access_stats(self, Ac: DeviceCsrCluster, B: DeviceCsr) -> AccessStats:
        st = L.bsp_access_stats()
        _check(self.lib.bsp_cluster_access_stats(self.h, C.byref(Ac.s), C.byref(B.s), C.byref(st)))
        return AccessStats(st.b_row_loads, st.a_inner_iters, st.placeholder_skips)

    def rowwise_access_stats(self, A: DeviceCsr, B: DeviceCsr) -> AccessStats:
        st = L.bsp_access_stats()
        _check(self.lib.bsp_rowwise_access_stats(self.h, C.byref(A.s), C.byref(B.s), C.byref(st)))
        return AccessStats(st.b_row_loads, st.a_inner_iters, st.placeholder_skips)

    # -- candidates ------------------------------------------------------------
    def _adopt_pairs(self, p, n) -> np.ndarray:
        cnt = int(n.value)
        out = np.zeros(cnt, dtype=CandidatePair)
        if cnt:
            raw = C.cast(p, C.POINTER(C.c_char * (cnt * CandidatePair.itemsize))).contents
            out = np.frombuffer(bytes(raw), dtype=CandidatePair).copy()
        self.lib.bsp_host_free_plain(C.cast(p, C.c_void_p))
        return out

    def spgemm_topk(self, A: DeviceCsr, At: DeviceCsr, topk: int, jacc_th: float) -> np.ndarray:
        p = C.POINTER(L.bsp_candidate)()
        n = C.c_int64()
        _check(self.lib.bsp_spgemm_topk(self.h, C.byref(A.s), C.byref(At.s), topk, jacc_th,
                                        C.byref(p), C.byref(n)))
        return self._adopt_pairs(p, n)

    def minhash_candidates(self, A: DeviceCsr, nhash: int = 64, bands: int = 32, seed: int = 1,
                           topk: int = 7, jacc_th: float = 0.3) -> np.ndarray:
        p = C.POINTER(L.bsp_candidate)()
        n = C.c_int64()
        _check(self.lib.bsp_minhash_candidates(self.h, C.byref(A.s), nhash, bands, seed, topk,
                                               jacc_th, C.byref(p), C.byref(n)))
        return self._adopt_pairs(p, n)

    def hierarchical_clusters(self, a: CsrMatrix, params: ClusterParams = ClusterParams(),
                              method: str = "topk", nhash: int = 64, bands: int = 32,
                              seed: int = 1) -> ClusterAssignment:
        ha = a._host()
        nc = C.c_int64()
        ptr = C.POINTER(C.c_int64)()
        rows = C.POINTER(C.c_int32)()
        m = {"topk": 0, "minhash": 1}[method]
        _check(self.lib.bsp_hierarchical_clusters(self.h, C.byref(ha), params.jacc_th,
                                                  params.max_cluster_th, m, nhash, bands, seed,
                                                  C.byref(nc), C.byref(ptr), C.byref(rows)))
        return ClusterAssignment._adopt(int(nc.value), ptr, rows)


_default: Optional[Engine] = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


# ---------------------------------------------------------------------------
# reference-shaped free functions (host in, host out)
# ---------------------------------------------------------------------------
def _dims(a: CsrMatrix, b: CsrMatrix) -> None:
    if a.ncols != b.nrows:
        raise ContractError("spgemm: dimension mismatch (a.ncols != b.nrows)")


def spgemm_rowwise(a: CsrMatrix, b: CsrMatrix, num_threads: int = 0) -> CsrMatrix:
    """reference spgemm.hpp:70-106 (num_threads accepted for signature parity)."""
    _dims(a, b)
    return default_engine().spgemm_rowwise_host(a, b)


def spgemm_symbolic(a: CsrMatrix, b: CsrMatrix, num_threads: int = 0) -> np.ndarray:
    """reference spgemm.hpp:41-63."""
    _dims(a, b)
    e = default_engine()
    A, B = e.upload(a), e.upload(b)
    return e.spgemm_symbolic(A, B)


def spgemm_topk(a: CsrMatrix, a_t: CsrMatrix, topk: int, jacc_th: float,
                num_threads: int = 0) -> np.ndarray:
    """reference spgemm.hpp:144-206; returns a CandidatePair record array."""
    if a.ncols != a_t.nrows:
        raise ContractError("spgemm_topk: dimension mismatch")
    if topk < 1:
        raise ContractError("spgemm_topk: topk must be >= 1")
    e = default_engine()
    return e.spgemm_topk(e.upload(a), e.upload(a_t), topk, jacc_th)


def jaccard_similarity(a: CsrMatrix, i: int, j: int) -> float:
    """reference spgemm.hpp:110-129."""
    out = C.c_double()
    ha = a._host()
    _check(L.load().bsp_jaccard(C.byref(ha), i, j, C.byref(out)))
    return float(out.value)


def build_csr_cluster(a: CsrMatrix, asg: ClusterAssignment) -> DeviceCsrCluster:
    """reference cluster_format.hpp:130-186 (device-resident result)."""
    e = default_engine()
    return e.build_csr_cluster(e.upload(a), asg)


def cluster_to_csr(m: DeviceCsrCluster) -> CsrMatrix:
    """reference cluster_format.hpp:190-233."""
    return m.engine.cluster_to_csr(m).download()


def spgemm_clusterwise(a: DeviceCsrCluster, b: CsrMatrix, num_threads: int = 0) -> CsrMatrix:
    """reference cluster_spgemm.hpp:186-189; C is returned as CSR over the
    original rows (equal to cluster_to_csr of the reference's result)."""
    if a.ncols != b.nrows:
        raise ContractError("spgemm_clusterwise: dimension mismatch (a.ncols != b.nrows)")
    e = a.engine
    return e.spgemm_clusterwise(a, e.upload(b)).download()


def spgemm_clusterwise_instrumented(a: DeviceCsrCluster, b: CsrMatrix, num_threads: int = 0):
    """reference cluster_spgemm.hpp:191-197: (C, AccessStats)."""
    e = a.engine
    B = e.upload(b)
    c = e.spgemm_clusterwise(a, B).download()
    return c, e.cluster_access_stats(a, B)


def rowwise_access_stats(a: CsrMatrix, b: CsrMatrix) -> AccessStats:
    """reference cluster_spgemm.hpp:34-45."""
    _dims(a, b)
    e = default_engine()
    return e.rowwise_access_stats(e.upload(a), e.upload(b))


def fixed_length_clusters(nrows: int, k: int) -> ClusterAssignment:
    """reference clustering.hpp:59-69."""
    nc, ptr, rows = C.c_int64(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    _check(L.load().bsp_fixed_length_clusters(nrows, k, C.byref(nc), C.byref(ptr), C.byref(rows)))
    return ClusterAssignment._adopt(int(nc.value), ptr, rows)


def variable_length_clusters(a: CsrMatrix, params: ClusterParams = ClusterParams()) -> ClusterAssignment:
    """reference clustering.hpp:76-93."""
    nc, ptr, rows = C.c_int64(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    ha = a._host()
    _check(L.load().bsp_variable_length_clusters(C.byref(ha), params.jacc_th, params.max_cluster_th,
                                                 C.byref(nc), C.byref(ptr), C.byref(rows)))
    return ClusterAssignment._adopt(int(nc.value), ptr, rows)


def hierarchical_clusters(a: CsrMatrix, params: ClusterParams = ClusterParams(),
                          num_threads: int = 0, method: str = "topk", **kw) -> ClusterAssignment:
    """reference clustering.hpp:109-185 (GPU candidates + host merge)."""
    return default_engine().hierarchical_clusters(a, params, method=method, **kw)


def merge_candidates(a: CsrMatrix, pairs: np.ndarray, params: ClusterParams = ClusterParams()):
    """Host heap/union-find merge over an external candidate list
    (reference clustering.hpp:122-183).  Returns (assignment, merge trace)."""
    pairs = np.ascontiguousarray(pairs, dtype=CandidatePair)
    nc, ptr, rows = C.c_int64(), C.POINTER(C.c_int64)(), C.POINTER(C.c_int32)()
    nm, mp = C.c_int64(), C.POINTER(L.bsp_candidate)()
    ha = a._host()
    _check(L.load().bsp_merge_candidates(C.byref(ha),
                                         C.cast(pairs.ctypes.data, C.POINTER(L.bsp_candidate)),
                                         pairs.size, params.jacc_th, params.max_cluster_th,
                                         C.byref(nc), C.byref(ptr), C.byref(rows), C.byref(nm),
                                         C.byref(mp)))
    asg = ClusterAssignment._adopt(int(nc.value), ptr, rows)
    trace = _adopt_pairs_plain(mp, nm)
    return asg, trace


def _adopt_pairs_plain(p, n) -> np.ndarray:
    cnt = int(n.value)
    out = np.zeros(cnt, dtype=CandidatePair)
    if cnt:
        raw = C.cast(p, C.POINTER(C.c_char * (cnt * CandidatePair.itemsize))).contents
        out = np.frombuffer(bytes(raw), dtype=CandidatePair).copy()
    L.load().bsp_host_free_plain(C.cast(p, C.c_void_p))
    return out


def assignment_to_permutation(asg: ClusterAssignment) -> Permutation:
    """reference clustering.hpp:189-194."""
    return Permutation.from_perm(asg.rows)


def reorder_random(nrows: int, seed: int) -> Permutation:
    """reference reorder.hpp:20-30 (identical permutation for a seed)."""
    p = np.empty(nrows, np.int32)
    _check(L.load().bsp_reorder_random(nrows, seed, _ptr(p)))
    return Permutation(p)


def reorder_degree(a: CsrMatrix) -> Permutation:
    """reference reorder.hpp:33-40."""
    p = np.empty(a.nrows, np.int32)
    ha = a._host()
    _check(L.load().bsp_reorder_degree(C.byref(ha), _ptr(p)))
    return Permutation(p)


def reorder_rcm(a: CsrMatrix) -> Permutation:
    """reference reorder.hpp:137-181 (identical permutation)."""
    p = np.empty(a.nrows, np.int32)
    ha = a._host()
    _check(L.load().bsp_reorder_rcm(C.byref(ha), _ptr(p)))
    return Permutation(p)


def bandwidth(a: CsrMatrix) -> int:
    """reference reorder.hpp:44-51."""
    out = C.c_int64()
    ha = a._host()
    _check(L.load().bsp_bandwidth(C.byref(ha), C.byref(out)))
    return int(out.value)


def generate_frontiers(a: CsrMatrix, num_frontiers: int = 10, batch: int = 64,
                       seed: int = 0) -> list:
    """reference frontier.hpp:20-77 (host CSR in, host CSRs out; BFS on the GPU)."""
    e = default_engine()
    A = e.upload(a)
    try:
        fs = e.generate_frontiers(A, num_frontiers, batch, seed)
        out = []
        for f in fs:
            out.append(f.download())
            f.free()
        return out
    finally:
        A.free()


def transpose(a: CsrMatrix) -> CsrMatrix:
    """reference csr.hpp:115-135."""
    ha, out = a._host(), L.bsp_host_csr()
    _check(L.load().bsp_transpose_host(C.byref(ha), C.byref(out)))
    return CsrMatrix._adopt(out)


def permute_symmetric(a: CsrMatrix, p: Permutation) -> CsrMatrix:
    """reference csr.hpp:146-172."""
    if a.nrows != a.ncols:
        raise ContractError("permute_symmetric: matrix must be square")
    if p.size != a.nrows:
        raise ContractError("permute_symmetric: permutation size mismatch")
    ha, out = a._host(), L.bsp_host_csr()
    _check(L.load().bsp_permute_symmetric(C.byref(ha), _ptr(p.perm), C.byref(out)))
    return CsrMatrix._adopt(out)


def permute_rows(a: CsrMatrix, p: Permutation) -> CsrMatrix:
    """reference csr.hpp:175-193."""
    if p.size != a.nrows:
        raise ContractError("permute_rows: permutation size mismatch")
    ha, out = a._host(), L.bsp_host_csr()
    _check(L.load().bsp_permute_rows(C.byref(ha), _ptr(p.perm), C.byref(out)))
    return CsrMatrix._adopt(out)


# ---------------------------------------------------------------------------
# file IO and reorder specs (reference matrix_market.hpp, reorder.hpp:183-192)
# ---------------------------------------------------------------------------
def load_matrix_market(path: str) -> CsrMatrix:
    """reference load_matrix_market + coo_to_csr (matrix_market.hpp:42-119)."""
    out = L.bsp_host_csr()
    _check(L.load().bsp_load_matrix_market(str(path).encode(), C.byref(out)))
    return CsrMatrix._adopt(out)


def write_matrix_market(a: CsrMatrix, path: str) -> None:
    """reference write_matrix_market (matrix_market.hpp:122-137)."""
    ha = a._host()
    _check(L.load().bsp_write_matrix_market(C.byref(ha), str(path).encode()))


def load_permutation(path: str, nrows: int) -> Permutation:
    """reference load_permutation (matrix_market.hpp:141-166)."""
    p = np.zeros(nrows, np.int32)
    _check(L.load().bsp_load_permutation(str(path).encode(), nrows, _ptr(p)))
    return Permutation.from_perm(p)


def write_permutation(p: Permutation, path: str) -> None:
    """reference write_permutation (matrix_market.hpp:168-173)."""
    perm = np.ascontiguousarray(p.perm, np.int32)
    _check(L.load().bsp_write_permutation(_ptr(perm), perm.size, str(path).encode()))


@dataclass
class ReorderSpec:
    """reference ReorderSpec (reorder.hpp:183-192): original, random (seed),
    degree, rcm, or an external permutation file (graph / hypergraph
    partitioning orders)."""
    method: str = "original"
    seed: int = 0
    path: str = ""

    def name(self) -> str:  # reference reorder_name (bench.hpp:51-59)
        return f"file:{self.path}" if self.method == "file" else self.method


def make_permutation(spec: ReorderSpec, a: CsrMatrix) -> Permutation:
    """reference detail::make_permutation (bench.hpp:119-127)."""
    if spec.method == "original":
        return Permutation.identity(a.nrows)
    if spec.method == "random":
        return reorder_random(a.nrows, spec.seed)
    if spec.method == "degree":
        return reorder_degree(a)
    if spec.method == "rcm":
        return reorder_rcm(a)
    if spec.method == "file":
        return load_permutation(spec.path, a.nrows)
    raise ContractError(f"unknown reorder method '{spec.method}'")


# ---------------------------------------------------------------------------
# seeded generators (BASELINE.json configs; recipes pinned in DESIGN.md)
# ---------------------------------------------------------------------------
def _gen(fn, *args) -> CsrMatrix:
    out = L.bsp_host_csr()
    _check(fn(*args, C.byref(out)))
    return CsrMatrix._adopt(out)


def gen_er(n: int, per_row: int, seed: int) -> CsrMatrix:
    return _gen(L.load().bsp_gen_er, n, per_row, seed)


def gen_hidden_clusters(ntemplates: int, children: int, tcols: int, keep_p: float,
                        extra_mean: float, seed: int, perm_seed: int) -> CsrMatrix:
    return _gen(L.load().bsp_gen_hidden_clusters, ntemplates, children, tcols, keep_p, extra_mean,
                seed, perm_seed)


def gen_rmat(scale: int, edge_factor: int, a: float, b: float, c: float, seed: int) -> CsrMatrix:
    return _gen(L.load().bsp_gen_rmat, scale, edge_factor, a, b, c, seed)


def gen_stencil27(g: int, perm_seed: int = -1) -> CsrMatrix:
    return _gen(L.load().bsp_gen_stencil27, g, perm_seed)


# BASELINE.json configs[0..4] with their pinned seeds.
CONFIGS = {
    1: dict(name="cfg1_er16384x8", kind="er", n=16384, per_row=8, seed=1),
    2: dict(name="cfg2_hidden_clusters_262144", kind="hidden", ntemplates=32768, children=8,
            tcols=16, keep_p=0.8, extra_mean=3.0, seed=2, perm_seed=22),
    3: dict(name="cfg3_rmat20_ef16", kind="rmat", scale=20, ef=16, a=0.57, b=0.19, c=0.19, seed=3),
    4: dict(name="cfg4_stencil27_128", kind="stencil", g=128, perm_seed=4),
    5: dict(name="cfg5_rmat22_ef8", kind="rmat", scale=22, ef=8, a=0.45, b=0.22, c=0.22, seed=5),
}


def make_config(cfg: int, scale_override: Optional[int] = None) -> CsrMatrix:
    """Generate BASELINE config `cfg` (1..5).  scale_override shrinks the R-MAT
    scale / grid / template count for fast parity tests of the same recipe."""
    c = CONFIGS[cfg]
    if c["kind"] == "er":
        return gen_er(c["n"] if scale_override is None else scale_override, c["per_row"], c["seed"])
    if c["kind"] == "hidden":
        nt = c["ntemplates"] if scale_override is None else scale_override
        return gen_hidden_clusters(nt, c["children"], c["tcols"], c["keep_p"], c["extra_mean"],
                                   c["seed"], c["perm_seed"])
    if c["kind"] == "rmat":
        sc = c["scale"] if scale_override is None else scale_override
        return gen_rmat(sc, c["ef"], c["a"], c["b"], c["c"], c["seed"])
    g = c["g"] if scale_override is None else scale_override
    return gen_stencil27(g, c["perm_seed"])
