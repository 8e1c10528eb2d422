"""ctypes binding of the C ABI (include/fuzzyclust_cuda.h).

This is the reference-side binding a Python caller would add.
The library is loaded from the in-tree ``lib/libfuzzyclust_cuda.so``; there is
no fallback: if it is missing or no B200 is visible, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref

import numpy as np

from .build import LIB
from .errors import DeviceError, raise_for

GPA, FISTA, FISTA_BT = 0, 1, 2
REASONS = {0: "tol_reached", 1: "max_iter", 2: "loss_increase_fista"}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


class SolverConfigC(C.Structure):
    _fields_ = [("step_size", C.c_double), ("max_iter", C.c_uint64), ("tol", C.c_double),
                ("method", C.c_int32), ("fista_restart", C.c_int32), ("trace_every", C.c_uint64),
                ("bt_eta", C.c_double), ("bt_max", C.c_uint32), ("flags", C.c_uint32)]


class TraceRecordC(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("loss", C.c_double), ("elapsed_ms", C.c_double),
                ("loss_increased", C.c_int32), ("backtracks", C.c_int32), ("step", C.c_double)]


class SummaryC(C.Structure):
    _fields_ = [("reason", C.c_int32), ("pad", C.c_int32), ("iterations", C.c_uint64),
                ("final_loss", C.c_double), ("step_size", C.c_double), ("n_records", C.c_uint64)]


class GraphSpecC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("blocks", C.c_uint32), ("n", C.c_uint64), ("m", C.c_uint64),
                ("seed", C.c_uint64), ("p_in", C.c_double), ("alpha", C.c_double), ("gamma", C.c_double),
                ("locality", C.c_int32), ("threads", C.c_int32)]


# every symbol include/fuzzyclust_cuda.h declares: (restype, argtypes)
class RefinePairsC(C.Structure):
    _fields_ = [("pairs", C.c_uint64), ("a_worst", C.c_double), ("a_index", C.c_uint64), ("a_col", C.c_uint32),
                ("a_plus", C.c_uint32), ("a_minus", C.c_uint32), ("pad0", C.c_uint32), ("b_worst", C.c_double),
                ("b_index", C.c_uint64), ("b_col", C.c_uint32), ("b_plus", C.c_uint32), ("b_minus", C.c_uint32),
                ("b_base_plus", C.c_uint32), ("b_base_minus", C.c_uint32), ("pad1", C.c_uint32)]


SIGNATURES = {
    "fc_version": (C.c_char_p, []),
    "fc_abi_version": (C.c_int, []),
    "fc_last_error": (C.c_char_p, [C.c_void_p]),
    "fc_nccl_unique_id": (C.c_int, [C.c_char_p]),
    "fc_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, C.c_char_p]),
    "fc_create_virtual": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int]),
    "fc_set_parity_mode": (C.c_int, [C.c_void_p, C.c_int]),
    "fc_get_parity_mode": (C.c_int, [C.c_void_p]),
    "fc_halo_info": (C.c_int, [C.c_void_p, _u64p, _u64p]),
    "fc_loopback_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_int]),
    "fc_loopback_destroy": (None, [C.c_void_p]),
    "fc_create_loopback": (C.c_int, [C.POINTER(C.c_void_p), C.c_void_p, C.c_int]),
    "fc_destroy": (None, [C.c_void_p]),
    "fc_upload_csr": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _i64p, _u32p, _dp, C.c_double]),
    "fc_partition": (C.c_int, [C.c_void_p, _u64p, C.c_int]),
    "fc_share_matrix": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp]),
    "fc_fused_column_pass": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, _dp]),
    "fc_loss_decomposed": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, _dp]),
    "fc_gpa_step_fused": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, _dp, C.c_double, _dp]),
    "fc_gpa_step": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, C.c_double, _dp]),
    "fc_project_simplex_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, _dp]),
    "fc_gradient_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, _dp, _dp, _dp, _dp]),
    "fc_loss_terms_rows": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint64, _dp, _dp, _dp]),
    "fc_solve": (C.c_int, [C.c_void_p, C.POINTER(SolverConfigC), C.c_uint32, _dp, _dp,
                           C.POINTER(TraceRecordC), C.c_uint64, C.POINTER(SummaryC)]),
    "fc_solver_begin": (C.c_int, [C.c_void_p, C.POINTER(SolverConfigC), C.c_uint32, _dp]),
    "fc_solver_run": (C.c_int, [C.c_void_p, C.c_uint64]),
    "fc_solver_sync": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "fc_solver_end": (C.c_int, [C.c_void_p, _dp, C.POINTER(TraceRecordC), C.c_uint64, C.POINTER(SummaryC)]),
    "fc_solver_finish": (C.c_int, [C.c_void_p, _dp, C.POINTER(TraceRecordC), C.c_uint64, C.POINTER(SummaryC)]),
    "fc_solver_checkpoint": (C.c_int, [C.c_void_p, C.c_char_p]),
    "fc_solver_resume": (C.c_int, [C.c_void_p, C.c_char_p]),
    "fc_stream": (C.c_void_p, [C.c_void_p]),
    "fc_launch_count": (C.c_uint64, [C.c_void_p]),
    "fc_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
    "fc_kernel_times": (C.c_int, [C.c_void_p, _dp, _u64p, C.c_int]),
    "fc_plan_partition": (C.c_int, [C.c_uint64, _i64p, C.c_int, _u64p]),
    "fc_generate_graph": (C.c_int, [C.POINTER(GraphSpecC), _u64p, C.POINTER(_i64p), C.POINTER(_u32p)]),
    "fc_build_from_triplets": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _u32p, _u32p, _dp, _i64p, _u32p, _dp,
                                         _dp, C.POINTER(C.c_int)]),
    "fc_build_similarity": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _u32p, _i64p, _u32p, _dp]),
    "fc_cross_share": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, _dp]),
    "fc_hessian_vector_product": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, _dp]),
    "fc_frob_inner": (C.c_double, [_dp, _dp, C.c_uint64]),
    "fc_refine_pairs": (C.c_int, [C.c_void_p, C.c_uint32, _dp, _dp, C.c_double, C.c_double, C.c_uint64, _u32p,
                                  C.c_uint64, C.POINTER(RefinePairsC)]),
    "fc_ingest_edge_list": (C.c_int, [C.c_void_p, C.c_char_p, C.c_uint64, C.c_int, C.c_void_p]),
    "fc_graph_lcc_nodes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _u32p, C.POINTER(_u32p),
                                     C.POINTER(C.c_uint64)]),
    "fc_graph_two_core_nodes": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _u32p, C.POINTER(_u32p),
                                          C.POINTER(C.c_uint64)]),
    "fc_free": (None, [C.c_void_p]),
}

KERNEL_CLASSES = ("step", "gram", "sweep", "rowsum", "combine", "finalize", "comm", "pack")

_lib = None


def lib():
    """Load the CUDA library (never a CPU substitute)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise DeviceError(f"CUDA library not built: {LIB} (run __graft_entry__.build())")
        L = C.CDLL(LIB)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a, t=_dp):
    return None if a is None else a.ctypes.data_as(t)


def _check(rc, ctx=None):
    if rc:
        raise_for(rc, lib().fc_last_error(ctx).decode())


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().fc_nccl_unique_id(buf))
    return buf.raw


def plan_partition(row_ptr, world: int):
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    out = np.zeros(world + 1, np.uint64)
    _check(lib().fc_plan_partition(rp.size - 1, _p(rp, _i64p), world, _p(out, _u64p)))
    return out


def generate_graph(kind: int, n: int, m: int, seed: int, *, blocks: int = 16, p_in: float = 0.9,
                   alpha: float = 2.5, gamma: float = 2.0, locality: bool = False, threads: int = 0):
    """Synthetic A+I CSR (host, multithreaded, deterministic). Returns (row_ptr, col_idx)."""
    spec = GraphSpecC(kind, blocks, n, m, seed, p_in, alpha, gamma, int(locality), threads)
    nnz = C.c_uint64()
    rp = _i64p()
    ci = _u32p()
    _check(lib().fc_generate_graph(C.byref(spec), C.byref(nnz), C.byref(rp), C.byref(ci)))
    try:
        row_ptr = np.ctypeslib.as_array(rp, shape=(n + 1,)).copy()
        col_idx = np.ctypeslib.as_array(ci, shape=(max(nnz.value, 1),))[: nnz.value].copy()
    finally:
        lib().fc_free(C.cast(rp, C.c_void_p))
        lib().fc_free(C.cast(ci, C.c_void_p))
    return row_ptr, col_idx


def frob_inner(a, b) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("frob_inner: shape mismatch")
    return float(lib().fc_frob_inner(_p(a), _p(b), a.size))


class IngestResultC(C.Structure):
    _fields_ = [("parsed_nodes", C.c_uint64), ("lcc_nodes", C.c_uint64), ("num_nodes", C.c_uint64),
                ("num_edges", C.c_uint64), ("edges", C.POINTER(C.c_uint32)), ("original_ids", C.POINTER(C.c_int64))]


def _take(ptr, count, dtype):
    """Copy `count` items out of a library-malloc'ed buffer and free it."""
    arr = np.ctypeslib.as_array(ptr, shape=(max(1, count),))[:count].astype(dtype, copy=True)
    lib().fc_free(C.cast(ptr, C.c_void_p))
    return arr


class LoopbackGroup:
    """fc_loopback: `world` rank contexts of ONE process on one device (one host thread
    per rank), exchanging through stream-ordered device copies instead of NCCL -- the
    multi-rank code path (shards, allgather, ordered chain, broadcast) without 8 GPUs."""

    def __init__(self, world: int, device: int = 0):
        h = C.c_void_p()
        rc = lib().fc_loopback_create(C.byref(h), device, world)
        if rc:
            raise_for(rc, lib().fc_last_error(None).decode())
        self.h, self.world, self.device = h, world, device

    def context(self, rank: int) -> "Context":
        return Context(self.device, rank=rank, world=self.world, loopback=self)

    def close(self):
        if getattr(self, "h", None):
            lib().fc_loopback_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """One device (one process per GPU).  world > 1: NCCL row-sharded solver
    (or, with `loopback`, one rank of an in-process LoopbackGroup)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None,
                 virtual_shards: int | None = None, loopback: "LoopbackGroup | None" = None):
        L = lib()
        h = C.c_void_p()
        if loopback is not None:
            rc = L.fc_create_loopback(C.byref(h), loopback.h, rank)
        elif virtual_shards:
            rc = L.fc_create_virtual(C.byref(h), device, virtual_shards)
        else:
            rc = L.fc_create(C.byref(h), device, rank, world, nccl_id)
        if rc:
            raise_for(rc, L.fc_last_error(None).decode())
        self.h = h
        self.device, self.rank, self.world = device, rank, world
        self.n = None

    def set_parity_mode(self, mode: int) -> None:
        """0 = bitwise (default), 1 = tolerance mode (see include/fuzzyclust_cuda.h)."""
        self._c(lib().fc_set_parity_mode(self.h, int(mode)))

    def parity_mode(self) -> int:
        return int(lib().fc_get_parity_mode(self.h))

    def halo_info(self):
        """(halo_mode, rows received per exchange, rows sent per exchange)."""
        r, s = C.c_uint64(), C.c_uint64()
        mode = lib().fc_halo_info(self.h, C.byref(r), C.byref(s))
        return int(mode), int(r.value), int(s.value)

    def close(self):
        if getattr(self, "h", None):
            lib().fc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _c(self, rc):
        if rc:
            raise_for(rc, lib().fc_last_error(self.h).decode())

    # ---- similarity ----------------------------------------------------------
    def upload(self, graph) -> None:
        self._c(lib().fc_upload_csr(self.h, graph.n, graph.nnz, _p(graph.row_ptr, _i64p),
                                    _p(graph.col_idx, _u32p), _p(graph.values), graph.frob_sq))
        self.n = graph.n
        try:
            self._graph_ref = weakref.ref(graph)
        except TypeError:
            self._graph_ref = None

    # ---- edge-list ingest (fc_ingest.cu) ---------------------------------------
    def ingest(self, text: bytes, stages: int = 2) -> dict:
        r = IngestResultC()
        self._c(lib().fc_ingest_edge_list(self.h, text, len(text), stages, C.byref(r)))
        edges = _take(r.edges, 2 * r.num_edges, np.uint32).reshape(-1, 2)
        ids = _take(r.original_ids, r.num_nodes, np.int64)
        return {"parsed_nodes": int(r.parsed_nodes), "lcc_nodes": int(r.lcc_nodes), "num_nodes": int(r.num_nodes),
                "edges": edges, "original_ids": ids}

    def _graph_nodes(self, fn, num_nodes, edges):
        e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        out = _u32p()
        cnt = C.c_uint64()
        self._c(fn(self.h, int(num_nodes), e.shape[0], _p(e, _u32p), C.byref(out), C.byref(cnt)))
        return _take(out, cnt.value, np.uint32)

    def lcc_nodes(self, num_nodes, edges):
        return self._graph_nodes(lib().fc_graph_lcc_nodes, num_nodes, edges)

    def two_core_nodes(self, num_nodes, edges):
        return self._graph_nodes(lib().fc_graph_two_core_nodes, num_nodes, edges)

    def refine_pairs(self, x, grad, eps_active, eps_grad_orth, budget, want_triples=False):
        x = np.ascontiguousarray(x, dtype=np.float64)
        grad = np.ascontiguousarray(grad, dtype=np.float64)
        r = RefinePairsC()
        cap = 0
        tri = None
        if want_triples:
            # count first (a cheap pass), then fetch the list
            self._c(lib().fc_refine_pairs(self.h, x.shape[1], _p(x), _p(grad), eps_active, eps_grad_orth, 0, None,
                                          0, C.byref(r)))
            cap = int(r.pairs)
            tri = np.empty((max(cap, 1), 3), np.uint32)
        self._c(lib().fc_refine_pairs(self.h, x.shape[1], _p(x), _p(grad), eps_active, eps_grad_orth,
                                      min(int(budget), 2**64 - 1), _p(tri, _u32p) if want_triples else None, cap,
                                      C.byref(r)))
        out = {f: getattr(r, f) for f, _ in RefinePairsC._fields_ if not f.startswith("pad")}
        out["triples"] = tri[:cap] if want_triples else None
        return out

    def cross_share(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        g = np.empty((a.shape[1], a.shape[1]))
        self._c(lib().fc_cross_share(self.h, a.shape[1], _p(a), _p(b), _p(g)))
        return g

    def hessian_vector_product(self, x, v):
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(x)
        self._c(lib().fc_hessian_vector_product(self.h, x.shape[1], _p(x), _p(v), _p(out)))
        return out

    def build_from_triplets(self, n, rows, cols, values=None):
        """fc_build_from_triplets: device from_triplets; the result is resident and returned."""
        from .similarity import SparseSimilarity
        rows = np.ascontiguousarray(rows, dtype=np.uint32)
        cols = np.ascontiguousarray(cols, dtype=np.uint32)
        nnz = rows.size
        vals = None if values is None else np.ascontiguousarray(values, dtype=np.float64)
        rp = np.empty(int(n) + 1, np.int64)
        ci = np.empty(nnz, np.uint32)
        vo = np.empty(nnz, np.float64) if vals is not None else None
        frob = C.c_double()
        pat = C.c_int()
        self._c(lib().fc_build_from_triplets(self.h, int(n), nnz, _p(rows, _u32p), _p(cols, _u32p), _p(vals),
                                             _p(rp, _i64p), _p(ci, _u32p), _p(vo), C.byref(frob), C.byref(pat)))
        s = SparseSimilarity(int(n), rp, ci, None if pat.value else vo, frob.value)
        self._adopt(s)
        return s

    def build_similarity(self, num_nodes, edges):
        """fc_build_similarity: device A + I from an (m, 2) edge list; resident and returned."""
        from .similarity import SparseSimilarity
        e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        nnz = int(num_nodes) + 2 * e.shape[0]
        rp = np.empty(int(num_nodes) + 1, np.int64)
        ci = np.empty(nnz, np.uint32)
        frob = C.c_double()
        self._c(lib().fc_build_similarity(self.h, int(num_nodes), e.shape[0], _p(e, _u32p), _p(rp, _i64p),
                                          _p(ci, _u32p), C.byref(frob)))
        s = SparseSimilarity(int(num_nodes), rp, ci, None, frob.value)
        self._adopt(s)
        return s

    def _adopt(self, graph):
        self.n = graph.n
        try:
            self._graph_ref = weakref.ref(graph)
        except TypeError:
            self._graph_ref = None

    def partition(self):
        out = np.zeros(65, np.uint64)
        parts = lib().fc_partition(self.h, _p(out, _u64p), 64)
        if parts < 0:
            self._c(2)
        return out[: parts + 1]

    # ---- granular operators (X is (N, C) row-major == the reference's C x N col-major)
    def share_matrix(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        c = x.shape[1]
        g = np.empty((c, c))
        self._c(lib().fc_share_matrix(self.h, c, _p(x), _p(g)))
        return g

    def fused_column_pass(self, x, want_xs: bool = True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        xs = np.empty_like(x) if want_xs else None
        m = C.c_double()
        self._c(lib().fc_fused_column_pass(self.h, x.shape[1], _p(x), _p(xs), C.byref(m)))
        return xs, m.value

    def loss_decomposed(self, x, g):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.ascontiguousarray(g, dtype=np.float64)
        v = C.c_double()
        self._c(lib().fc_loss_decomposed(self.h, x.shape[1], _p(x), _p(g), C.byref(v)))
        return v.value

    def gpa_step_fused(self, x, g, xs, tau):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._c(lib().fc_gpa_step_fused(self.h, x.shape[1], _p(x), _p(np.ascontiguousarray(g, dtype=np.float64)),
                                        _p(np.ascontiguousarray(xs, dtype=np.float64)), tau, _p(out)))
        return out

    def gpa_step(self, x, g, tau):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._c(lib().fc_gpa_step(self.h, x.shape[1], _p(x), _p(np.ascontiguousarray(g, dtype=np.float64)), tau,
                                  _p(out)))
        return out

    def project_simplex_rows(self, x):
        y = np.array(x, dtype=np.float64, copy=True, order="C")
        if y.ndim == 1:
            y = y.reshape(1, -1)
        self._c(lib().fc_project_simplex_rows(self.h, y.shape[1], y.shape[0], _p(y)))
        return y

    def gradient_rows(self, g, xs, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        x2 = x.reshape(-1, x.shape[-1])
        out = np.empty_like(x2)
        self._c(lib().fc_gradient_rows(self.h, x2.shape[1], x2.shape[0], _p(np.ascontiguousarray(g, dtype=np.float64)),
                                       _p(np.ascontiguousarray(xs, dtype=np.float64).reshape(x2.shape)), _p(x2), _p(out)))
        return out.reshape(x.shape)

    def loss_terms_rows(self, xs, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        x2 = x.reshape(-1, x.shape[-1])
        out = np.empty(x2.shape[0])
        self._c(lib().fc_loss_terms_rows(self.h, x2.shape[1], x2.shape[0],
                                         _p(np.ascontiguousarray(xs, dtype=np.float64).reshape(x2.shape)), _p(x2), _p(out)))
        return out

    # ---- solver -------------------------------------------------------------
    @staticmethod
    def config(method=GPA, step_size=0.0, max_iter=100000, tol=0.0, trace_every=1, fista_restart=False,
               bt_eta=2.0, bt_max=30):
        return SolverConfigC(step_size, max_iter, tol, method, int(fista_restart), trace_every, bt_eta, bt_max, 0)

    def solve(self, x0, cfg: SolverConfigC, want_x: bool = True, trace_cap: int | None = None, out=None):
        """fc_solve.  `out`: optional preallocated (n, c) float64 result buffer (e.g. a
        page-locked one, which the library fills by direct DMA)."""
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        n, c = x0.shape
        cap = trace_cap if trace_cap is not None else int(min(cfg.max_iter + 2, 1 << 20))
        recs = (TraceRecordC * max(cap, 1))()
        summ = SummaryC()
        if want_x:
            if out is None:
                out = np.empty_like(x0)
            elif out.shape != x0.shape or out.dtype != np.float64 or not out.flags.c_contiguous:
                raise ValueError("solve: out must be a C-contiguous float64 array shaped like x0")
        else:
            out = None
        self._c(lib().fc_solve(self.h, C.byref(cfg), c, _p(x0), _p(out), recs, cap, C.byref(summ)))
        return _result(out, recs, summ, cap)

    def begin(self, x0, cfg: SolverConfigC):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        self._cfg = cfg
        self._c(lib().fc_solver_begin(self.h, C.byref(cfg), x0.shape[1], _p(x0)))

    def run(self, iterations: int):
        self._c(lib().fc_solver_run(self.h, iterations))

    def sync(self) -> bool:
        d = C.c_int()
        self._c(lib().fc_solver_sync(self.h, C.byref(d)))
        return bool(d.value)

    def end(self, n, c, want_x=True, trace_cap=None):
        cap = trace_cap if trace_cap is not None else int(min(self._cfg.max_iter + 2, 1 << 20))
        recs = (TraceRecordC * max(cap, 1))()
        summ = SummaryC()
        out = np.empty((n, c)) if want_x else None
        self._c(lib().fc_solver_end(self.h, _p(out), recs, cap, C.byref(summ)))
        return _result(out, recs, summ, cap)

    def finish(self, n, c, want_x=True, trace_cap=None):
        """fc_solver_finish: run the remaining iterations of the session, then end()."""
        cap = trace_cap if trace_cap is not None else int(min(self._cfg.max_iter + 2, 1 << 20))
        recs = (TraceRecordC * max(cap, 1))()
        summ = SummaryC()
        out = np.empty((n, c)) if want_x else None
        self._c(lib().fc_solver_finish(self.h, _p(out), recs, cap, C.byref(summ)))
        return _result(out, recs, summ, cap)

    def checkpoint(self, path):
        """fc_solver_checkpoint: save the running session to `path`."""
        self._c(lib().fc_solver_checkpoint(self.h, os.fsencode(path)))

    def resume(self, path, cfg: SolverConfigC):
        """fc_solver_resume: reopen a saved session (cfg: the run's config, for trace sizing)."""
        self._cfg = cfg
        self._c(lib().fc_solver_resume(self.h, os.fsencode(path)))

    # ---- instrumentation ----------------------------------------------------
    def stream_ptr(self) -> int:
        return lib().fc_stream(self.h) or 0

    def launch_count(self) -> int:
        return int(lib().fc_launch_count(self.h))

    def set_profiling(self, on: bool):
        self._c(lib().fc_set_profiling(self.h, int(on)))

    def kernel_times(self):
        ms = np.zeros(len(KERNEL_CLASSES))
        n = np.zeros(len(KERNEL_CLASSES), np.uint64)
        self._c(lib().fc_kernel_times(self.h, _p(ms), _p(n, _u64p), len(KERNEL_CLASSES)))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KERNEL_CLASSES)}


def _result(out, recs, summ, cap):
    k = min(summ.n_records, cap)
    return {
        "membership": out,
        "reason": REASONS[summ.reason],
        "iterations": int(summ.iterations),
        "final_loss": summ.final_loss,
        "step_size": summ.step_size,
        "records": [(int(recs[i].iteration), recs[i].loss, bool(recs[i].loss_increased)) for i in range(k)],
        "elapsed_ms": [recs[i].elapsed_ms for i in range(k)],
        "backtracks": [int(recs[i].backtracks) for i in range(k)],
        "steps": [recs[i].step for i in range(k)],
        "n_records": int(summ.n_records),
    }
