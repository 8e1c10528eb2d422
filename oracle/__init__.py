"""TEST INFRASTRUCTURE ONLY -- ctypes access to the CPU checkers.

* ``Oracle``    -> oracle/_build/libfcoracle.so : plain-C restatement (fc_oracle.c)
* ``Reference`` -> oracle/_ref/libfcref.so     : the unmodified reference headers
                                                 behind ref_driver.cpp

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_2506_04045_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libfcoracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfcref.so")

GPA, FISTA, FISTA_BT = 0, 1, 2
REASONS = {0: "tol_reached", 1: "max_iter", 2: "loss_increase_fista"}

_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)


def build() -> None:
    """Compile both checkers (the reference one only when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None else None


class _Csr(C.Structure):
    _fields_ = [("n", C.c_uint64), ("nnz", C.c_uint64), ("row_ptr", _i64p), ("col_idx", _u32p),
                ("values", _dp), ("frob_sq", C.c_double)]


class _Cfg(C.Structure):
    _fields_ = [("step_size", C.c_double), ("max_iter", C.c_uint64), ("tol", C.c_double),
                ("method", C.c_int), ("trace_every", C.c_uint64), ("fista_restart", C.c_int),
                ("bt_eta", C.c_double), ("bt_max", C.c_uint32)]


class _Rec(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("loss", C.c_double), ("loss_increased", C.c_int32),
                ("backtracks", C.c_int32), ("step", C.c_double)]


class _Sum(C.Structure):
    _fields_ = [("reason", C.c_int32), ("pad", C.c_int32), ("iterations", C.c_uint64),
                ("final_loss", C.c_double), ("step_size", C.c_double), ("n_records", C.c_uint64)]


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


class Oracle:
    """The plain-C restatement.  Arrays are numpy; X is (N, C) row-major (== C x N col-major)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        L.fco_last_error.restype = C.c_char_p
        L.fco_splitmix_next.restype = C.c_uint64
        L.fco_splitmix_next.argtypes = [C.POINTER(C.c_uint64)]
        L.fco_project_simplex.argtypes = [_dp, C.c_size_t]
        L.fco_init_random.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, _dp]
        L.fco_feasibility_error.restype = C.c_double
        L.fco_feasibility_error.argtypes = [_dp, C.c_size_t, C.c_size_t]
        L.fco_share_matrix.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp]
        L.fco_share_frob_sq.restype = C.c_double
        L.fco_share_frob_sq.argtypes = [_dp, C.c_size_t]
        L.fco_cross_share.argtypes = [_dp, _dp, C.c_size_t, C.c_size_t, _dp]
        L.fco_hessian_vector_product.argtypes = [_dp, _dp, C.c_size_t, C.c_void_p, _dp]
        L.fco_frob_inner.restype = C.c_double
        L.fco_frob_inner.argtypes = [_dp, _dp, C.c_size_t]
        L.fco_fused_column_pass.argtypes = [_dp, C.c_size_t, C.POINTER(_Csr), _dp, _dp]
        L.fco_loss_decomposed.restype = C.c_double
        L.fco_loss_decomposed.argtypes = [_dp, C.c_size_t, C.POINTER(_Csr), _dp]
        L.fco_gpa_step_fused.argtypes = [_dp, C.c_size_t, C.c_size_t, _dp, _dp, C.c_double, _dp]
        L.fco_fista_t_next.restype = C.c_double
        L.fco_fista_t_next.argtypes = [C.c_double]
        L.fco_default_step_size.restype = C.c_double
        L.fco_default_step_size.argtypes = [C.POINTER(_Csr), C.c_size_t]
        L.fco_solve.argtypes = [C.POINTER(_Csr), C.POINTER(_Cfg), C.c_size_t, _dp, _dp,
                                C.POINTER(_Rec), C.c_uint64, C.POINTER(_Sum)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.fco_last_error().decode())

    @staticmethod
    def csr(g) -> _Csr:
        s = _Csr(g.n, g.nnz, _ptr(g.row_ptr, _i64p), _ptr(g.col_idx, _u32p),
                 _ptr(g.values), g.frob_sq)
        s._keep = g
        return s

    def splitmix_stream(self, seed: int, count: int):
        st = C.c_uint64(seed)
        return [self.lib.fco_splitmix_next(C.byref(st)) for _ in range(count)]

    def project_simplex(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        self._check(self.lib.fco_project_simplex(_ptr(y), y.size))
        return y

    def init_random(self, n, c, seed):
        x = np.empty((n, c))
        self._check(self.lib.fco_init_random(n, c, seed, _ptr(x)))
        return x

    def feasibility_error(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return self.lib.fco_feasibility_error(_ptr(x), x.shape[1], x.shape[0])

    def share_matrix(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.empty((x.shape[1], x.shape[1]))
        self.lib.fco_share_matrix(_ptr(x), x.shape[1], x.shape[0], _ptr(g))
        return g

    def share_frob_sq(self, g):
        g = np.ascontiguousarray(g, dtype=np.float64)
        return self.lib.fco_share_frob_sq(_ptr(g), g.shape[0])

    def cross_share(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        g = np.empty((a.shape[1], a.shape[1]))
        self.lib.fco_cross_share(_ptr(a), _ptr(b), a.shape[1], a.shape[0], _ptr(g))
        return g

    def hessian_vector_product(self, x, v, graph):
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(x)
        s = self.csr(graph)
        self._check(self.lib.fco_hessian_vector_product(_ptr(x), _ptr(v), x.shape[1], C.byref(s), _ptr(out)))
        return out

    def frob_inner(self, a, b):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        return self.lib.fco_frob_inner(_ptr(a), _ptr(b), a.size)

    def fused_column_pass(self, x, graph):
        x = np.ascontiguousarray(x, dtype=np.float64)
        xs = np.empty_like(x)
        m = C.c_double()
        s = self.csr(graph)
        self._check(self.lib.fco_fused_column_pass(_ptr(x), x.shape[1], C.byref(s), _ptr(xs), C.byref(m)))
        return xs, m.value

    def loss_decomposed(self, x, graph, g):
        x = np.ascontiguousarray(x, dtype=np.float64)
        s = self.csr(graph)
        return self.lib.fco_loss_decomposed(_ptr(x), x.shape[1], C.byref(s), _ptr(np.ascontiguousarray(g)))

    def gpa_step_fused(self, x, g, xs, tau):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self.lib.fco_gpa_step_fused(_ptr(x), x.shape[1], x.shape[0], _ptr(np.ascontiguousarray(g)),
                                                _ptr(np.ascontiguousarray(xs)), tau, _ptr(out)))
        return out

    def fista_t_next(self, t):
        return self.lib.fco_fista_t_next(t)

    def default_step_size(self, graph):
        s = self.csr(graph)
        return self.lib.fco_default_step_size(C.byref(s), graph.n)

    def solve(self, graph, x0, *, method=GPA, step_size=0.0, max_iter=100000, tol=0.0, trace_every=1,
              fista_restart=False, bt_eta=2.0, bt_max=50):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        n, c = x0.shape
        cfg = _Cfg(step_size, max_iter, tol, method, trace_every, int(fista_restart), bt_eta, bt_max)
        cap = max_iter + 2
        recs = (_Rec * cap)()
        summ = _Sum()
        out = np.empty_like(x0)
        s = self.csr(graph)
        self._check(self.lib.fco_solve(C.byref(s), C.byref(cfg), c, _ptr(x0), _ptr(out), recs, cap,
                                       C.byref(summ)))
        k = min(summ.n_records, cap)
        return {
            "membership": out,
            "reason": REASONS[summ.reason],
            "iterations": summ.iterations,
            "final_loss": summ.final_loss,
            "step_size": summ.step_size,
            "records": [(recs[i].iteration, recs[i].loss, bool(recs[i].loss_increased)) for i in range(k)],
            "backtracks": [recs[i].backtracks for i in range(k)],
            "steps": [recs[i].step for i in range(k)],
        }


class _RRec(C.Structure):
    _fields_ = [("iteration", C.c_uint64), ("loss", C.c_double), ("loss_increased", C.c_int32),
                ("pad", C.c_int32), ("elapsed_ms", C.c_double)]


class _RSum(C.Structure):
    _fields_ = [("reason", C.c_int32), ("pad", C.c_int32), ("iterations", C.c_uint64),
                ("final_loss", C.c_double), ("step_size", C.c_double), ("n_records", C.c_uint64),
                ("solve_ms", C.c_double)]


GEN_SO = os.path.join(HERE, "_build", "libfcgen.so")


class _GraphSpec(C.Structure):   # include/fuzzyclust_cuda.h fc_graph_spec
    _fields_ = [("kind", C.c_int32), ("blocks", C.c_uint32), ("n", C.c_uint64), ("m", C.c_uint64),
                ("seed", C.c_uint64), ("p_in", C.c_double), ("alpha", C.c_double), ("gamma", C.c_double),
                ("locality", C.c_int32), ("threads", C.c_int32)]


class HostGraph:
    """A+I CSR on the host (all values 1.0): what the reference arm feeds oracle/_ref."""

    def __init__(self, n, row_ptr, col_idx):
        self.n, self.row_ptr, self.col_idx, self.values = int(n), row_ptr, col_idx, None
        self.nnz = int(col_idx.size)
        self.frob_sq = float(self.nnz)


def generate_graph(kind, n, m, seed, *, blocks=16, p_in=0.9, alpha=2.5, gamma=2.0, locality=False, threads=0):
    """The repo's synthetic generator (csrc/generator.cpp) built host-only (oracle/_build/libfcgen.so):
    the same graph ``paper_2506_04045_b200.generate_{sbm,citation}`` returns, without the CUDA library."""
    if not os.path.exists(GEN_SO):
        build()
    L = C.CDLL(GEN_SO)
    L.fcgen_generate.argtypes = [C.POINTER(_GraphSpec), C.POINTER(C.c_uint64), C.POINTER(_i64p),
                                 C.POINTER(_u32p), C.c_char_p, C.c_size_t]
    L.fcgen_free.argtypes = [C.c_void_p]
    spec = _GraphSpec(kind, blocks, n, m, seed, p_in, alpha, gamma, int(locality), threads)
    nnz = C.c_uint64()
    rp, ci = _i64p(), _u32p()
    err = C.create_string_buffer(512)
    rc = L.fcgen_generate(C.byref(spec), C.byref(nnz), C.byref(rp), C.byref(ci), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    try:
        row_ptr = np.ctypeslib.as_array(rp, shape=(n + 1,)).copy()
        col_idx = np.ctypeslib.as_array(ci, shape=(max(nnz.value, 1),))[: nnz.value].copy()
    finally:
        L.fcgen_free(C.cast(rp, C.c_void_p))
        L.fcgen_free(C.cast(ci, C.c_void_p))
    return HostGraph(n, row_ptr, col_idx)


def reference_available(path: str = REF_SO) -> bool:
    return os.path.exists(path)


class Reference:
    """The real reference library (unmodified headers) behind oracle/ref_driver.cpp."""

    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        L.fcref_last_error.restype = C.c_char_p
        L.fcref_resolve_workers.restype = C.c_uint
        L.fcref_similarity_create.argtypes = [C.c_uint64, C.c_uint64, _i64p, _u32p, _dp, C.c_int,
                                              C.POINTER(C.c_void_p)]
        L.fcref_similarity_free.argtypes = [C.c_void_p]
        L.fcref_similarity_frob_sq.restype = C.c_double
        L.fcref_similarity_frob_sq.argtypes = [C.c_void_p]
        L.fcref_similarity_nnz.restype = C.c_uint64
        L.fcref_similarity_nnz.argtypes = [C.c_void_p]
        L.fcref_similarity_export.argtypes = [C.c_void_p, _i64p, _u32p, _dp]
        L.fcref_from_triplets.argtypes = [C.c_uint64, C.c_uint64, _u32p, _u32p, _dp, C.POINTER(C.c_void_p)]
        L.fcref_build_similarity.argtypes = [C.c_uint64, C.c_uint64, _u32p, C.POINTER(C.c_void_p)]
        L.fcref_project_simplex.argtypes = [_dp, C.c_uint64]
        L.fcref_splitmix.restype = C.c_uint64
        L.fcref_splitmix.argtypes = [C.c_uint64, C.c_uint64]
        L.fcref_init_membership.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64, _dp]
        L.fcref_share_matrix.argtypes = [_dp, C.c_uint64, C.c_uint64, C.c_uint, _dp]
        L.fcref_fused_column_pass.argtypes = [C.c_void_p, _dp, C.c_uint64, C.c_uint, _dp, _dp]
        L.fcref_loss_decomposed.argtypes = [C.c_void_p, _dp, C.c_uint64, C.c_uint, _dp]
        L.fcref_load_pipeline.argtypes = [C.c_char_p, C.c_uint64, C.c_int, C.POINTER(C.c_uint64),
                                          C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                          C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.POINTER(C.c_int64))]
        L.fcref_graph_nodes.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint32), C.c_int,
                                        C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(C.c_uint64)]
        L.fcref_free_buf.argtypes = [C.c_void_p]
        L.fcref_refine.argtypes = [C.c_void_p, _dp, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                   C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int),
                                   C.POINTER(C.c_uint64), C.POINTER(_RVerdict), C.POINTER(_RVerdict), _dp, _dp, _dp]
        L.fcref_cross_share.argtypes = [_dp, _dp, C.c_uint64, C.c_uint64, C.c_uint, _dp]
        L.fcref_hessian_vector_product.argtypes = [C.c_void_p, _dp, _dp, C.c_uint64, C.c_uint, _dp, _dp]
        L.fcref_gpa_step_fused.argtypes = [_dp, C.c_uint64, C.c_uint64, _dp, _dp, C.c_double, C.c_uint, _dp]
        L.fcref_default_step_size.restype = C.c_double
        L.fcref_default_step_size.argtypes = [C.c_void_p]
        L.fcref_fista_t_next.restype = C.c_double
        L.fcref_fista_t_next.argtypes = [C.c_double]
        L.fcref_solve.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_double, C.c_int, C.c_uint64,
                                  C.c_int, C.c_uint, C.c_uint64, _dp, _dp, C.POINTER(_RRec), C.c_uint64,
                                  C.POINTER(_RSum)]

    def _check(self, rc):
        if rc:
            raise OracleError(rc, self.lib.fcref_last_error().decode())

    def similarity(self, graph, fast=False):
        h = C.c_void_p()
        self._check(self.lib.fcref_similarity_create(graph.n, graph.nnz, _ptr(graph.row_ptr, _i64p),
                                                     _ptr(graph.col_idx, _u32p), _ptr(graph.values),
                                                     int(fast), C.byref(h)))
        return RefSimilarity(self, h)

    def from_triplets(self, n, rows, cols, values):
        """sparse.hpp:28-62 on triplets in the given order (uint32 indices, float64 values)."""
        r = np.ascontiguousarray(rows, dtype=np.uint32)
        c = np.ascontiguousarray(cols, dtype=np.uint32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        h = C.c_void_p()
        self._check(self.lib.fcref_from_triplets(n, r.size, _ptr(r, _u32p), _ptr(c, _u32p), _ptr(v),
                                                 C.byref(h)))
        return RefSimilarity(self, h)

    def build_similarity(self, num_nodes, edges):
        e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1, 2)
        h = C.c_void_p()
        self._check(self.lib.fcref_build_similarity(num_nodes, e.shape[0], _ptr(e, _u32p), C.byref(h)))
        return RefSimilarity(self, h)

    def project_simplex(self, x):
        y = np.array(x, dtype=np.float64, copy=True)
        self._check(self.lib.fcref_project_simplex(_ptr(y), y.size))
        return y

    def splitmix(self, seed, k):
        return self.lib.fcref_splitmix(seed, k)

    def init_membership(self, n, c, kind=0, seed=0, row=0):
        out = np.empty((n, c))
        self._check(self.lib.fcref_init_membership(n, c, kind, seed, row, _ptr(out)))
        return out

    def share_matrix(self, x, workers=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        g = np.empty((x.shape[1], x.shape[1]))
        self._check(self.lib.fcref_share_matrix(_ptr(x), x.shape[1], x.shape[0], workers, _ptr(g)))
        return g

    def load_pipeline(self, text: bytes, stages: int = 2):
        """(parsed_nodes, lcc_nodes, num_nodes, edges (m, 2) uint32, original_ids) of the reference."""
        pn, ln, nn, ne = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        e = C.POINTER(C.c_uint32)()
        ids = C.POINTER(C.c_int64)()
        self._check(self.lib.fcref_load_pipeline(text, len(text), stages, C.byref(pn), C.byref(ln), C.byref(nn),
                                                 C.byref(ne), C.byref(e), C.byref(ids)))
        edges = np.ctypeslib.as_array(e, shape=(max(1, 2 * ne.value),))[: 2 * ne.value].copy().reshape(-1, 2)
        orig = np.ctypeslib.as_array(ids, shape=(max(1, nn.value),))[: nn.value].copy()
        self.lib.fcref_free_buf(C.cast(e, C.c_void_p))
        self.lib.fcref_free_buf(C.cast(ids, C.c_void_p))
        return pn.value, ln.value, nn.value, edges, orig

    def graph_nodes(self, n, edges, which):
        """which 0: largest_connected_component_nodes, 1: two_core_nodes."""
        e = np.ascontiguousarray(edges, dtype=np.uint32).reshape(-1)
        out = C.POINTER(C.c_uint32)()
        cnt = C.c_uint64()
        self._check(self.lib.fcref_graph_nodes(n, e.size // 2, e.ctypes.data_as(C.POINTER(C.c_uint32)), which,
                                               C.byref(out), C.byref(cnt)))
        v = np.ctypeslib.as_array(out, shape=(max(1, cnt.value),))[: cnt.value].copy()
        self.lib.fcref_free_buf(C.cast(out, C.c_void_p))
        return v

    def cross_share(self, a, b, workers=1):
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        g = np.empty((a.shape[1], a.shape[1]))
        self._check(self.lib.fcref_cross_share(_ptr(a), _ptr(b), a.shape[1], a.shape[0], workers, _ptr(g)))
        return g

    def gpa_step_fused(self, x, g, xs, tau, workers=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self.lib.fcref_gpa_step_fused(_ptr(x), x.shape[1], x.shape[0],
                                                  _ptr(np.ascontiguousarray(g)), _ptr(np.ascontiguousarray(xs)),
                                                  tau, workers, _ptr(out)))
        return out

    def fista_t_next(self, t):
        return self.lib.fcref_fista_t_next(t)


class _RVerdict(C.Structure):
    _fields_ = [("status", C.c_int), ("has_witness", C.c_int), ("has_base", C.c_int),
                ("interior_shortcut", C.c_int), ("tested", C.c_uint64), ("value", C.c_double)]


class RefSimilarity:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h

    def __del__(self):
        try:
            self.ref.lib.fcref_similarity_free(self.h)
        except Exception:
            pass

    @property
    def frob_sq(self):
        return self.ref.lib.fcref_similarity_frob_sq(self.h)

    @property
    def nnz(self):
        return self.ref.lib.fcref_similarity_nnz(self.h)

    def export(self, n):
        nnz = self.nnz
        rp = np.empty(n + 1, np.int64)
        ci = np.empty(nnz, np.uint32)
        v = np.empty(nnz)
        self.ref._check(self.ref.lib.fcref_similarity_export(self.h, _ptr(rp, _i64p), _ptr(ci, _u32p), _ptr(v)))
        return rp, ci, v

    def default_step_size(self):
        return self.ref.lib.fcref_default_step_size(self.h)

    def fused_column_pass(self, x, workers=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        xs = np.empty_like(x)
        m = C.c_double()
        self.ref._check(self.ref.lib.fcref_fused_column_pass(self.h, _ptr(x), x.shape[1], workers, _ptr(xs),
                                                             C.byref(m)))
        return xs, m.value

    def refine(self, x, tau_probe=1e-2, eps_critical=1e-2, eps_active=1e-8, eps_grad_orth=1e-6, eps_quad=1e-8,
               eps_cone=1e-9, random_directions=0, seed=0, budget=2**64 - 1):
        """secondorder.hpp refine() of the reference: a dict of the report, dense witnesses."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        crit, st = C.c_int(), C.c_int()
        res = C.c_double()
        gen = C.c_uint64()
        a, b = _RVerdict(), _RVerdict()
        wa, wb, wbase = np.zeros_like(x), np.zeros_like(x), np.zeros_like(x)
        self.ref._check(self.ref.lib.fcref_refine(
            self.h, _ptr(x), x.shape[1], tau_probe, eps_critical, eps_active, eps_grad_orth, eps_quad, eps_cone,
            random_directions, seed, budget, C.byref(crit), C.byref(res), C.byref(st), C.byref(gen), C.byref(a),
            C.byref(b), _ptr(wa), _ptr(wb), _ptr(wbase)))
        ver = lambda v, w, base: {"status": v.status, "tested": v.tested, "value": v.value,
                                  "interior_shortcut": bool(v.interior_shortcut),
                                  "witness": w if v.has_witness else None, "base": base if v.has_base else None}
        return {"critical": bool(crit.value), "residual": res.value, "status": st.value,
                "directions_generated": gen.value, "a": ver(a, wa, None), "b": ver(b, wb, wbase)}

    def hessian_vector_product(self, x, v, workers=1):
        """(HVP, quadratic_form) of the reference (objective.hpp:186-223)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(x)
        q = C.c_double()
        self.ref._check(self.ref.lib.fcref_hessian_vector_product(self.h, _ptr(x), _ptr(v), x.shape[1], workers,
                                                                  _ptr(out), C.byref(q)))
        return out, q.value

    def loss_decomposed(self, x, workers=1):
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = C.c_double()
        self.ref._check(self.ref.lib.fcref_loss_decomposed(self.h, _ptr(x), x.shape[1], workers, C.byref(v)))
        return v.value

    def solve(self, x0, *, method=GPA, step_size=0.0, max_iter=100000, tol=0.0, trace_every=1,
              fista_restart=False, workers=1, want_x=True):
        x0 = np.ascontiguousarray(x0, dtype=np.float64)
        n, c = x0.shape
        cap = max_iter + 2
        recs = (_RRec * cap)()
        summ = _RSum()
        out = np.empty_like(x0) if want_x else None
        self.ref._check(self.ref.lib.fcref_solve(self.h, step_size, max_iter, tol, method, trace_every,
                                                 int(fista_restart), workers, c, _ptr(x0), _ptr(out), recs, cap,
                                                 C.byref(summ)))
        k = min(summ.n_records, cap)
        return {
            "membership": out,
            "reason": REASONS[summ.reason],
            "iterations": summ.iterations,
            "final_loss": summ.final_loss,
            "step_size": summ.step_size,
            "records": [(recs[i].iteration, recs[i].loss, bool(recs[i].loss_increased)) for i in range(k)],
            "elapsed_ms": [recs[i].elapsed_ms for i in range(k)],
            "solve_ms": summ.solve_ms,
        }
