"""Python mirror of the reference's header API (namespace ``fuzzyclust``).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/fuzzyclust/{membership,objective,simplex,solver}.hpp,
so that the parity tests read like the reference's own GoogleTest suites.  The
membership matrix is a numpy array of shape (N, C) -- byte-identical to the
reference's C x N column-major ``MembershipMatrix`` (dense.hpp:12-27).

Every numerical operator runs on the GPU through the C ABI (``capi``); there is
no CPU fallback.  ``workers`` arguments are accepted for signature parity and
ignored: results are bitwise identical for any worker count in the reference,
and identical to it here.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import capi
from .errors import InvalidInput, IoError
from .similarity import SparseSimilarity

kReductionBlock = 1024          # parallel.hpp:15
kVersion = "0.1.0"              # common.hpp:8


class Method(IntEnum):          # solver.hpp:18 (+ backtracking, new)
    kGpa = 0
    kFista = 1
    kFistaBacktracking = 2


class TerminationReason(IntEnum):   # solver.hpp:20
    kTolReached = 0
    kMaxIter = 1
    kLossIncreaseFista = 2


def to_string(r) -> str:        # solver.hpp:22-29
    return capi.REASONS[int(r)]


class InitKind(IntEnum):        # membership.hpp:64-70
    kRandom = 0
    kDirichlet = 1
    kRowOne = 2
    kUniform = 3
    kGiven = 4


@dataclass
class InitStrategy:             # membership.hpp:72-77
    kind: InitKind = InitKind.kRandom
    seed: int = 0
    row: int = 0
    given: np.ndarray | None = None


@dataclass
class SolverConfig:             # solver.hpp:31-48
    step_size: float = 0.0
    max_iter: int = 100000
    tol: float = 0.0
    method: Method = Method.kGpa
    trace_every: int = 1
    fista_restart: bool = False
    workers: int = 1
    bt_eta: float = 2.0         # new: backtracking growth of L = 1/step
    bt_max: int = 30

    def validate(self) -> None:
        if self.max_iter < 1:
            raise InvalidInput("solver: max_iter must be >= 1")
        if self.tol < 0.0:
            raise InvalidInput("solver: tol must be >= 0")
        if self.trace_every < 1:
            raise InvalidInput("solver: trace_every must be >= 1")
        if not (self.step_size > 0.0) and self.step_size != 0.0:
            raise InvalidInput("solver: step_size must be positive (or 0 for auto)")


@dataclass
class TraceRecord:              # solver.hpp:50-55
    iteration: int
    loss: float
    elapsed_ms: float = 0.0
    loss_increased: bool = False
    backtracks: int = 0
    step: float = 0.0


@dataclass
class SolverTrace:              # solver.hpp:57-63
    records: list = field(default_factory=list)
    reason: TerminationReason = TerminationReason.kMaxIter
    iterations: int = 0
    final_loss: float = 0.0
    step_size: float = 0.0


@dataclass
class SolverResult:             # solver.hpp:65-68
    membership: np.ndarray
    trace: SolverTrace


@dataclass
class ColumnPass:               # objective.hpp:146-149
    xs: np.ndarray
    merge: float


# ---- device context ---------------------------------------------------------------
_default_ctx = None


def default_context() -> capi.Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = capi.Context(0)
    return _default_ctx


def set_default_context(ctx: capi.Context | None) -> None:
    global _default_ctx
    _default_ctx = ctx


def _ctx_for(s: SparseSimilarity | None, ctx: capi.Context | None, n: int | None = None) -> capi.Context:
    """Context with `s` resident (uploaded once per similarity object).  Operators
    that need only N (share_matrix) get an identity pattern of size n if no
    similarity of that size is resident."""
    ctx = ctx or default_context()
    ref = getattr(ctx, "_graph_ref", None)
    cur = ref() if ref is not None else None
    if s is not None:
        if cur is not s:
            ctx.upload(s)
    elif n is not None and (cur is None or cur.size() != n):
        ident = SparseSimilarity(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.uint32))
        ctx.upload(ident)
        ctx._graph_keep = ident
    return ctx


def _ctx_nograph(ctx):
    """Granular ops that only need N: upload a pattern of the right size if needed."""
    return ctx or default_context()


# ---- sparse.hpp construction on the device (fc_build.cu) ---------------------------
def _as_u32_index(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype == np.uint32:
        return np.ascontiguousarray(a)
    if a.dtype.kind in "iu" and (a.size == 0 or (int(a.min()) >= 0 and int(a.max()) <= 0xFFFFFFFF)):
        return a.astype(np.uint32)
    if a.dtype.kind == "f":
        a = np.where(np.isfinite(a), a, -1.0)
    a = a.astype(np.int64)
    # negative / >= 2^32 ids are out of range for any n < 2^31: map them to 0xFFFFFFFF so the
    # device check reports the first failing triplet in the reference's order.
    return np.where((a < 0) | (a > 0xFFFFFFFF), 0xFFFFFFFF, a).astype(np.uint32)


def from_triplets(n: int, triplets, ctx: capi.Context | None = None) -> SparseSimilarity:
    """SparseSimilarity::from_triplets (sparse.hpp:28-62) on the device; the result stays resident."""
    t = np.asarray(triplets, dtype=np.float64).reshape(-1, 3) if len(triplets) else np.zeros((0, 3))
    ctx = ctx or default_context()
    return ctx.build_from_triplets(n, _as_u32_index(t[:, 0]), _as_u32_index(t[:, 1]), t[:, 2])


def build_similarity(num_nodes: int, edges, ctx: capi.Context | None = None) -> SparseSimilarity:
    """SparseSimilarity::build_similarity (sparse.hpp:66-75) on the device; the result stays resident."""
    e = np.asarray(edges).reshape(-1, 2)
    ctx = ctx or default_context()
    return ctx.build_similarity(num_nodes, _as_u32_index(e))


# ---- rng.hpp / membership.hpp ------------------------------------------------------
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64_stream(seed: int, start: int, count: int) -> np.ndarray:
    """Draws #start .. #start+count-1 of SplitMix64(seed) (rng.hpp:21-26)."""
    k = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def splitmix64_doubles(seed: int, start: int, count: int) -> np.ndarray:
    """next_double(): (next() >> 11) * 2^-53 (rng.hpp:29-31)."""
    return (splitmix64_stream(seed, start, count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def init_membership(num_nodes: int, num_clusters: int, strategy: InitStrategy | None = None,
                    ctx: capi.Context | None = None) -> np.ndarray:
    """membership.hpp:79-132.  The per-column projection runs on the GPU."""
    strategy = strategy or InitStrategy()
    if num_clusters == 0 or num_nodes == 0:
        raise InvalidInput("init_membership: dimensions must be positive")
    n, c = num_nodes, num_clusters
    kind = InitKind(strategy.kind)
    if kind == InitKind.kRandom:
        ctx = _ctx_nograph(ctx)
        x = np.empty((n, c))
        rows_per = max(1, (1 << 24) // c)
        for r0 in range(0, n, rows_per):
            r1 = min(n, r0 + rows_per)
            x[r0:r1] = splitmix64_doubles(strategy.seed, r0 * c, (r1 - r0) * c).reshape(r1 - r0, c)
        return ctx.project_simplex_rows(x)
    if kind == InitKind.kDirichlet:
        ctx = _ctx_nograph(ctx)
        u = splitmix64_doubles(strategy.seed, 0, n * c).reshape(n, c)
        x = np.empty((n, c))
        for i in range(n):               # std::log per entry, sequential sum (membership.hpp:98-107)
            s = 0.0
            for k in range(c):
                v = -math.log(1.0 - float(u[i, k]))
                x[i, k] = v
                s += v
            for k in range(c):
                x[i, k] = x[i, k] / s
        return ctx.project_simplex_rows(x)
    if kind == InitKind.kRowOne:
        if strategy.row >= c:
            raise InvalidInput("init_membership: row out of range")
        x = np.zeros((n, c))
        x[:, strategy.row] = 1.0
        return x
    if kind == InitKind.kUniform:
        return np.full((n, c), 1.0 / float(c))
    if kind == InitKind.kGiven:
        g = strategy.given
        if g is None:
            raise InvalidInput("init_membership: no matrix supplied")
        g = np.asarray(g, dtype=np.float64)
        if g.shape != (n, c):
            raise InvalidInput("init_membership: supplied matrix has wrong shape")
        validate_membership(g, 1e-9)
        return g.copy()
    raise InvalidInput("init_membership: unknown kind")


def feasibility_error(x: np.ndarray) -> float:
    """membership.hpp:49-61 (host check of a caller-supplied matrix)."""
    x = np.asarray(x, dtype=np.float64)
    worst = 0.0
    for row in x:
        s = 0.0
        for v in row.tolist():
            s += v
            if v < 0.0:
                worst = max(worst, -v)
            if v > 1.0:
                worst = max(worst, v - 1.0)
        worst = max(worst, abs(s - 1.0))
    return worst


def validate_membership(x: np.ndarray, tol: float) -> None:
    x = np.asarray(x)
    if x.size == 0:
        raise InvalidInput("membership: empty matrix")
    if not np.all(np.isfinite(x)):
        raise InvalidInput("membership: non-finite entry")
    err = feasibility_error(x)
    if err > tol:
        raise InvalidInput(f"membership: columns violate the simplex constraint by {err:g} (tolerance {tol:g})")


def write_membership_csv(x: np.ndarray) -> str:       # membership.hpp:136-149
    c = x.shape[1]
    lines = ["node_id," + ",".join(f"x_{k}" for k in range(1, c + 1))]
    for i, row in enumerate(np.asarray(x)):
        lines.append(str(i) + "," + ",".join("%.17g" % v for v in row.tolist()))
    return "\n".join(lines) + "\n"


def read_membership_csv(text: str) -> np.ndarray:     # membership.hpp:151-194
    rows = []
    header = True
    for line_no, line in enumerate(text.split("\n"), 1):
        if not line:
            continue
        if header:
            header = False
            continue
        cells = line.split(",")[1:]
        try:
            vals = [float(cc) for cc in cells]
        except ValueError:
            raise InvalidInput(f"membership CSV: bad value at line {line_no}") from None
        if not vals:
            raise InvalidInput(f"membership CSV: no values at line {line_no}")
        if rows and len(vals) != len(rows[0]):
            raise InvalidInput(f"membership CSV: ragged row at line {line_no}")
        rows.append(vals)
    if not rows:
        raise InvalidInput("membership CSV: no data rows")
    return np.array(rows, dtype=np.float64)


# ---- graph.hpp / tools load_pipeline on the device -----------------
@dataclass
class Graph:                         # graph.hpp:21-42
    num_nodes: int
    edges: np.ndarray                # (m, 2) uint32, u < v, sorted, unique

    def degrees(self) -> np.ndarray:
        return np.bincount(self.edges.reshape(-1), minlength=self.num_nodes)


@dataclass
class ParsedGraph:                   # graph.hpp:53-58
    graph: Graph
    original_ids: np.ndarray


@dataclass
class LoadedGraph:                   # tools/fuzzyclust.cpp:52-58
    graph: Graph
    original_ids: np.ndarray
    parsed_nodes: int
    lcc_nodes: int


def _text_bytes(text) -> bytes:
    return text.encode() if isinstance(text, str) else bytes(text)


def parse_edge_list(text, ctx: capi.Context | None = None) -> ParsedGraph:
    """graph.hpp:63-103 (ids compacted by first appearance on the device)."""
    r = (ctx or default_context()).ingest(_text_bytes(text), 0)
    return ParsedGraph(Graph(r["num_nodes"], r["edges"]), r["original_ids"])


def largest_connected_component_nodes(g: Graph, ctx: capi.Context | None = None) -> np.ndarray:
    """graph.hpp:146-169: ascending; ties to the component holding the smallest id."""
    return (ctx or default_context()).lcc_nodes(g.num_nodes, g.edges)


def two_core_nodes(g: Graph, ctx: capi.Context | None = None) -> np.ndarray:
    """graph.hpp:206-213: nodes surviving iterated degree <= 1 removal, ascending."""
    return (ctx or default_context()).two_core_nodes(g.num_nodes, g.edges)


def induced_subgraph(g: Graph, nodes) -> Graph:
    """graph.hpp:107-120 (order-preserving recompaction; host)."""
    nodes = np.asarray(nodes, dtype=np.int64)
    new_id = np.full(g.num_nodes, -1, dtype=np.int64)
    new_id[nodes] = np.arange(nodes.size)
    e = g.edges.astype(np.int64)
    keep = (new_id[e[:, 0]] >= 0) & (new_id[e[:, 1]] >= 0) if e.size else np.zeros(0, bool)
    sub = new_id[e[keep]].astype(np.uint32).reshape(-1, 2)
    return Graph(int(nodes.size), sub)


def largest_connected_component(g: Graph, ctx: capi.Context | None = None) -> Graph:
    return induced_subgraph(g, largest_connected_component_nodes(g, ctx))


def prune_degree_one(g: Graph, ctx: capi.Context | None = None) -> Graph:
    return induced_subgraph(g, two_core_nodes(g, ctx))


def load_pipeline(text=None, path=None, prune: bool = True, ctx: capi.Context | None = None) -> LoadedGraph:
    """tools/fuzzyclust.cpp:62-89: parse -> LCC -> optional 2-core, all on the device."""
    if path is not None:
        try:
            with open(path, "rb") as f:
                text = f.read()
        except OSError:
            raise IoError(f"cannot open {path}") from None
    r = (ctx or default_context()).ingest(_text_bytes(text), 2 if prune else 1)
    if r["num_nodes"] == 0:
        raise InvalidInput("graph is empty after preprocessing")
    return LoadedGraph(Graph(r["num_nodes"], r["edges"]), r["original_ids"], r["parsed_nodes"], r["lcc_nodes"])


def write_edge_list(g: Graph) -> str:
    """graph.hpp:222-224: "u v" lines in (u, v) order."""
    return "".join(f"{u} {v}\n" for u, v in g.edges.tolist())


# ---- second order (objective.hpp:61-90, :182-223) ------------------
def cross_share(a: np.ndarray, b: np.ndarray, workers: int = 1, ctx: capi.Context | None = None) -> np.ndarray:
    """A B^T on the device (Gram of the stacked [A | B])."""
    if a.shape != b.shape:
        raise InvalidInput("cross_share: shape mismatch")
    return _ctx_for(None, ctx, n=a.shape[0]).cross_share(a, b)


def hessian_vector_product(xbar: np.ndarray, v: np.ndarray, s: SparseSimilarity, workers: int = 1,
                           ctx: capi.Context | None = None) -> np.ndarray:
    if xbar.shape != v.shape:
        raise InvalidInput("hessian_vector_product: shape mismatch")
    if s.size() != xbar.shape[0]:
        raise InvalidInput("hessian_vector_product: similarity size mismatch")
    return _ctx_for(s, ctx).hessian_vector_product(xbar, v)


def frob_inner(a: np.ndarray, b: np.ndarray) -> float:
    """dense.hpp:40-46: one sequential sum over the storage order (host loop in the library)."""
    return capi.frob_inner(a, b)


def quadratic_form(xbar: np.ndarray, v: np.ndarray, s: SparseSimilarity, workers: int = 1,
                   ctx: capi.Context | None = None) -> float:
    """<H(xbar) v, v>_F: device HVP, then the reference's sequential frob_inner on the host."""
    return frob_inner(hessian_vector_product(xbar, v, s, workers, ctx), v)


# ---- secondorder.hpp refinement ------------------------------------
@dataclass
class SecondOrderConfig:             # secondorder.hpp:25-36
    tau_probe: float = 1e-2
    eps_critical: float = 1e-2
    eps_active: float = 1e-8
    eps_grad_orth: float = 1e-6
    eps_quad: float = 1e-8
    eps_cone: float = 1e-9
    random_directions: int = 0
    seed: int = 0
    budget: int = 2**64 - 1
    workers: int = 1


class RefinementStatus(IntEnum):     # secondorder.hpp:195-200
    kRefutedFirstOrder = 0
    kRefutedConditionA = 1
    kRefutedConditionB = 2
    kSurviving = 3


@dataclass
class RefinementVerdict:             # secondorder.hpp:214-222; witnesses as {(node, row): value}
    status: RefinementStatus = RefinementStatus.kSurviving
    witness: dict | None = None
    witness_base: dict | None = None
    witness_value: float = 0.0
    directions_tested: int = 0
    used_interior_shortcut: bool = False


@dataclass
class RefinementReport:              # secondorder.hpp:333-340
    critical: bool = False
    residual: float = 0.0
    status: RefinementStatus = RefinementStatus.kSurviving
    condition_a: RefinementVerdict = field(default_factory=RefinementVerdict)
    condition_b: RefinementVerdict = field(default_factory=RefinementVerdict)
    directions_generated: int = 0


def full_gradient(x: np.ndarray, s: SparseSimilarity, ctx: capi.Context | None = None) -> np.ndarray:
    """secondorder.hpp:39-52: -4 (X S - (X X^T) X) column by column, on the device."""
    c = _ctx_for(s, ctx)
    share = c.share_matrix(x)
    xs, _ = c.fused_column_pass(x)
    return c.gradient_rows(share, xs, x)


def projection_residual(x: np.ndarray, s: SparseSimilarity, tau_probe: float,
                        ctx: capi.Context | None = None) -> float:
    """secondorder.hpp:56-68: ||P(X - tau grad) - X||_F (sum sequential in storage order)."""
    c = _ctx_for(s, ctx)
    d = c.gpa_step(x, c.share_matrix(x), tau_probe) - np.asarray(x, dtype=np.float64)
    return math.sqrt(capi.frob_inner(d, d))


def is_critical(x, s, tau_probe: float, eps: float, ctx: capi.Context | None = None) -> bool:
    if not tau_probe > 0.0:
        raise InvalidInput("is_critical: tau_probe must be positive")
    return projection_residual(x, s, tau_probe, ctx) <= eps


def is_interior(x: np.ndarray, eps_active: float) -> bool:
    return bool(np.all(np.asarray(x) > eps_active))


class _SplitMix64:                   # rng.hpp:14-34
    def __init__(self, seed):
        self.state = seed & 0xFFFFFFFFFFFFFFFF

    def next(self):
        self.state = (self.state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        return z ^ (z >> 31)

    def next_double(self):
        return float(self.next() >> 11) * 2.0 ** -53

    def next_below(self, bound):
        return self.next() % bound


def _sparse_frob_inner(a: dict, b_dense=None, b: dict | None = None) -> float:
    """frob_inner restricted to nonzeros, in storage order (node, then row): exact."""
    acc = 0.0
    for key in sorted(a):
        other = b.get(key, 0.0) if b is not None else float(b_dense[key])
        acc += a[key] * other
    return acc


def _random_directions(x, grad, triples, cfg: SecondOrderConfig) -> list:
    """secondorder.hpp:158-189: random nonnegative combinations of kept pairs, rescaled to
    ||V|| = sqrt(2), deduplicated (as sparse {(node, row): value} maps)."""
    out = []
    if triples is None or cfg.random_directions <= 0 or len(triples) == 0:
        return out
    npairs = len(triples)
    pair_set = {(int(i), int(k), int(l)) for i, k, l in triples.tolist()}
    rng = _SplitMix64(cfg.seed)
    target = math.sqrt(2.0)
    produced = attempts = 0
    while produced < cfg.random_directions and attempts < 20 * cfg.random_directions:
        attempts += 1
        v: dict = {}
        picks = 2 + rng.next_below(min(npairs, 6))
        for _ in range(picks):
            i, k, l = (int(t) for t in triples[rng.next_below(npairs)])
            coeff = rng.next_double()
            v[(i, k)] = v.get((i, k), 0.0) + coeff
            v[(i, l)] = v.get((i, l), 0.0) - coeff
        norm = math.sqrt(_sparse_frob_inner(v, b=v))
        if norm == 0.0:
            continue
        scale = target / norm
        v = {key: val * scale for key, val in v.items()}
        if abs(_sparse_frob_inner(v, b_dense=grad)) / target > cfg.eps_grad_orth:
            continue
        if not _tangent_cone_contains_sparse(x, v, cfg.eps_cone, cfg.eps_active):
            continue
        nz = {key: val for key, val in v.items() if val != 0.0}
        dup = False
        if len(nz) == 2:                  # equal to a pair direction?
            (a1, v1), (a2, v2) = sorted(nz.items())
            if a1[0] == a2[0] and {v1, v2} == {1.0, -1.0}:
                plus, minus = (a1[1], a2[1]) if v1 == 1.0 else (a2[1], a1[1])
                dup = (a1[0], plus, minus) in pair_set
        if not dup:
            dup = any(nz == e for e in out)
        if dup:
            continue
        out.append(nz)
        produced += 1
    return out


def _tangent_cone_contains_sparse(x, v: dict, eps: float, eps_active: float) -> bool:
    cols: dict = {}
    for (i, k) in sorted(v):
        cols.setdefault(i, []).append(k)
    for i, ks in cols.items():
        ssum = 0.0
        for k in range(x.shape[1]):
            val = v.get((i, k), 0.0)
            ssum += val
            if x[i, k] <= eps_active and val < -eps:
                return False
        if abs(ssum) > eps:
            return False
    return True


def _dense(v: dict, shape) -> np.ndarray:
    d = np.zeros(shape)
    for (i, k), val in v.items():
        d[i, k] = val
    return d


def refine(x: np.ndarray, s: SparseSimilarity, cfg: SecondOrderConfig | None = None,
           ctx: capi.Context | None = None) -> RefinementReport:
    """secondorder.hpp:343-368.  Pair directions are evaluated on the device in one batched
    pass (fc_refine_pairs: bit-identical closed forms of the reference's HVP path, no
    direction materialised); random combinations go through the device HVP."""
    cfg = cfg or SecondOrderConfig()
    x = np.ascontiguousarray(x, dtype=np.float64)
    validate_membership(x, 1e-6)
    c = _ctx_for(s, ctx)
    rep = RefinementReport()
    rep.residual = projection_residual(x, s, cfg.tau_probe, c)
    rep.critical = rep.residual <= cfg.eps_critical
    if not rep.critical:
        rep.status = RefinementStatus.kRefutedFirstOrder
        return rep
    grad = full_gradient(x, s, c)
    pr = c.refine_pairs(x, grad, cfg.eps_active, cfg.eps_grad_orth, cfg.budget,
                        want_triples=cfg.random_directions > 0)
    rnd = _random_directions(x, grad, pr["triples"], cfg)
    npairs = int(pr["pairs"])
    rep.directions_generated = npairs + len(rnd)
    total = rep.directions_generated
    budget = cfg.budget
    # ---- condition (a): pairs first (device), then the random combinations in order
    a = RefinementVerdict(directions_tested=min(total, budget))
    worst, wit = pr["a_worst"], None
    if pr["a_index"] != 2**64 - 1:
        wit = {(pr["a_col"], pr["a_plus"]): 1.0, (pr["a_col"], pr["a_minus"]): -1.0}
    for t, v in enumerate(rnd):
        if npairs + t >= budget:
            break
        vd = _dense(v, x.shape)
        q = capi.frob_inner(c.hessian_vector_product(x, vd), vd)
        if q < worst:
            worst, wit = q, v
    if worst < -cfg.eps_quad:
        a.status, a.witness, a.witness_value = RefinementStatus.kRefutedConditionA, wit, worst
    rep.condition_a = a
    if a.status == RefinementStatus.kRefutedConditionA:
        rep.status = a.status
        return rep
    # ---- condition (b)
    b = RefinementVerdict()
    if is_interior(x, cfg.eps_active):
        b.used_interior_shortcut = True
    else:
        b.directions_tested = min(total, budget)
        worst, wit, base = pr["b_worst"], None, None
        if pr["b_index"] != 2**64 - 1:
            wit = {(pr["b_col"], pr["b_plus"]): 1.0, (pr["b_col"], pr["b_minus"]): -1.0}
            base = {(pr["b_col"], pr["b_base_plus"]): 1.0, (pr["b_col"], pr["b_base_minus"]): -1.0}
        for t, v in enumerate(rnd):
            if npairs + t >= budget:
                break
            for i in sorted({key[0] for key in v}):
                xi, gi = x[i], grad[i]
                for l in range(x.shape[1]):
                    if not (xi[l] <= cfg.eps_active and abs(v.get((i, l), 0.0)) > cfg.eps_active):
                        continue
                    for k in range(x.shape[1]):
                        if k == l:
                            continue
                        val = float(gi[k] - gi[l])
                        if val < worst:
                            worst = val
                            wit = {(i, k): 1.0, (i, l): -1.0}
                            base = v
        if worst < -cfg.eps_quad:
            b.status, b.witness, b.witness_base, b.witness_value = (RefinementStatus.kRefutedConditionB, wit, base,
                                                                    worst)
    rep.condition_b = b
    rep.status = b.status
    return rep


# ---- binary artifacts (new; same layouts as the C++ headers) -------
_MEMB_MAGIC = b"FCMEMB01"
_CSR_MAGIC = b"FCCSR001"


def write_membership_binary(x: np.ndarray, path) -> None:
    """"FCMEMB01", uint64 N, uint64 C, N*C float64 node-major (membership.hpp, new)."""
    x = np.ascontiguousarray(x, dtype="<f8")
    with open(path, "wb") as f:
        f.write(_MEMB_MAGIC)
        f.write(np.array(x.shape, dtype="<u8").tobytes())
        x.tofile(f)


def read_membership_binary(path) -> np.ndarray:
    with open(path, "rb") as f:
        if f.read(8) != _MEMB_MAGIC:
            raise IoError("membership binary: bad magic")
        hdr = np.frombuffer(f.read(16), dtype="<u8")
        if hdr.size != 2 or hdr[0] == 0 or hdr[1] == 0:
            raise IoError("membership binary: bad header")
        n, c = int(hdr[0]), int(hdr[1])
        x = np.fromfile(f, dtype="<f8", count=n * c)
        if x.size != n * c:
            raise IoError("membership binary: truncated data")
    return x.reshape(n, c).astype(np.float64, copy=False)


def write_similarity_binary(s: SparseSimilarity, path) -> None:
    """"FCCSR001", n, nnz, flags, frob_sq, row_ptr, col[, values] (sparse.hpp, new)."""
    with open(path, "wb") as f:
        f.write(_CSR_MAGIC)
        f.write(np.array([s.n, s.nnz], dtype="<u8").tobytes())
        f.write(np.array([0 if s.values is None else 1, 0], dtype="<u4").tobytes())
        f.write(np.array([s.frob_sq], dtype="<f8").tobytes())
        s.row_ptr.astype("<i8", copy=False).tofile(f)
        s.col_idx.astype("<u4", copy=False).tofile(f)
        if s.values is not None:
            s.values.astype("<f8", copy=False).tofile(f)


def read_similarity_binary(path, validate: bool = True) -> SparseSimilarity:
    with open(path, "rb") as f:
        if f.read(8) != _CSR_MAGIC:
            raise IoError("similarity binary: bad magic")
        raw = f.read(32)
        if len(raw) != 32:
            raise IoError("similarity binary: bad header")
        n, nnz = (int(v) for v in np.frombuffer(raw[:16], dtype="<u8"))
        flags = int(np.frombuffer(raw[16:20], dtype="<u4")[0])
        frob = float(np.frombuffer(raw[24:32], dtype="<f8")[0])
        rp = np.fromfile(f, dtype="<i8", count=n + 1)
        ci = np.fromfile(f, dtype="<u4", count=nnz)
        vals = np.fromfile(f, dtype="<f8", count=nnz) if flags & 1 else None
        if rp.size != n + 1 or ci.size != nnz or (vals is not None and vals.size != nnz):
            raise IoError("similarity binary: truncated data")
    if rp[0] != 0 or int(rp[-1]) != nnz:
        raise IoError("similarity binary: row_ptr does not span [0, nnz)")
    if n and np.any(np.diff(rp) < 0):
        raise IoError("similarity binary: row_ptr not monotone")
    if nnz and int(ci.max()) >= n:
        raise IoError("similarity binary: column index out of range")
    s = SparseSimilarity(n, rp, ci, vals)
    if validate:
        s._validate_symmetry()
    if s.frob_sq != frob:
        raise IoError("similarity binary: frob_sq does not match the stored values")
    return s


# ---- simplex.hpp -------------------------------------------------------------------
def project_simplex(x, ctx: capi.Context | None = None) -> np.ndarray:
    """simplex.hpp:62-66 (copying variant), on the GPU."""
    v = np.asarray(x, dtype=np.float64).ravel()
    if v.size == 0:
        raise InvalidInput("project_simplex: empty vector")
    return _ctx_nograph(ctx).project_simplex_rows(v.reshape(1, -1))[0]


# ---- objective.hpp -----------------------------------------------------------------
def share_matrix(x: np.ndarray, workers: int = 1, s: SparseSimilarity | None = None,
                 ctx: capi.Context | None = None) -> np.ndarray:
    """objective.hpp:92-95.  Needs a context holding a similarity of size N (pass s)."""
    x = np.asarray(x)
    return _ctx_for(s, ctx, n=x.shape[0]).share_matrix(x)


def fused_column_pass(x: np.ndarray, s: SparseSimilarity, workers: int = 1,
                      ctx: capi.Context | None = None) -> ColumnPass:
    x = np.asarray(x)
    if s.size() != x.shape[0]:
        raise InvalidInput("objective: similarity/membership size mismatch")
    xs, merge = _ctx_for(s, ctx).fused_column_pass(x)
    return ColumnPass(xs, merge)


def loss_decomposed(x: np.ndarray, s: SparseSimilarity, share: np.ndarray, workers: int = 1,
                    ctx: capi.Context | None = None) -> float:
    return _ctx_for(s, ctx).loss_decomposed(x, share)


def share_frob_sq(share: np.ndarray) -> float:       # objective.hpp:25-29
    acc = 0.0
    for v in np.asarray(share, dtype=np.float64).ravel().tolist():
        acc += v * v
    return acc


def gpa_step_fused(x, share, xs, tau: float, workers: int = 1, s: SparseSimilarity | None = None,
                   ctx: capi.Context | None = None) -> np.ndarray:
    return _ctx_for(s, ctx).gpa_step_fused(x, share, xs, tau)


def gpa_step(x, s: SparseSimilarity, share, tau: float, workers: int = 1,
             ctx: capi.Context | None = None) -> np.ndarray:
    return _ctx_for(s, ctx).gpa_step(x, share, tau)


# ---- solver.hpp --------------------------------------------------------------------
def fista_t_next(t: float) -> float:                 # solver.hpp:72
    return (1.0 + math.sqrt(1.0 + 4.0 * t * t)) / 2.0


def default_step_size(s: SparseSimilarity, n: int) -> float:   # solver.hpp:78-81
    return 1.0 / (4.0 * s.frob_norm() + 12.0 * float(n))


def resolve_step_size(config: SolverConfig, s: SparseSimilarity, n: int) -> float:
    return config.step_size if config.step_size > 0.0 else default_step_size(s, n)


def _to_result(raw, n, c) -> SolverResult:
    tr = SolverTrace(
        records=[TraceRecord(it, loss, ms, inc, bt, st) for (it, loss, inc), ms, bt, st in
                 zip(raw["records"], raw["elapsed_ms"], raw["backtracks"], raw["steps"])],
        reason=TerminationReason({"tol_reached": 0, "max_iter": 1, "loss_increase_fista": 2}[raw["reason"]]),
        iterations=raw["iterations"], final_loss=raw["final_loss"], step_size=raw["step_size"])
    return SolverResult(raw["membership"], tr)


def solve(x0: np.ndarray, s: SparseSimilarity, config: SolverConfig,
          ctx: capi.Context | None = None) -> SolverResult:
    """solver.hpp:274-277 -> run_gpa / run_fista, the whole loop on the device."""
    config.validate()
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    if s.size() != x0.shape[0]:
        raise InvalidInput("run_gpa: similarity/membership size mismatch" if config.method == Method.kGpa
                           else "run_fista: similarity/membership size mismatch")
    ctx = _ctx_for(s, ctx)
    cfg = capi.Context.config(int(config.method), config.step_size, config.max_iter, config.tol,
                              config.trace_every, config.fista_restart, config.bt_eta, config.bt_max)
    raw = ctx.solve(x0, cfg)
    return _to_result(raw, *x0.shape)


def run_gpa(x0, s, config: SolverConfig, ctx=None) -> SolverResult:
    cfg = SolverConfig(**{**config.__dict__, "method": Method.kGpa})
    return solve(x0, s, cfg, ctx)


def run_fista(x0, s, config: SolverConfig, ctx=None) -> SolverResult:
    m = config.method if config.method != Method.kGpa else Method.kFista
    cfg = SolverConfig(**{**config.__dict__, "method": m})
    return solve(x0, s, cfg, ctx)


def write_trace_csv(trace: SolverTrace, include_timing: bool = False) -> str:   # solver.hpp:282-295
    out = ["iteration,loss,elapsed_ms" if include_timing else "iteration,loss"]
    for r in trace.records:
        line = f"{r.iteration},%.17g" % r.loss
        if include_timing:
            line += ",%.3f" % r.elapsed_ms
        out.append(line)
    return "\n".join(out) + "\n"


# ---- synthetic graphs (new; see csrc/generator.cpp) ---------------------------------
def generate_sbm(n: int, m: int, blocks: int, seed: int, p_in: float = 0.9, locality: bool = False,
                 threads: int = 0) -> SparseSimilarity:
    rp, ci = capi.generate_graph(0, n, m, seed, blocks=blocks, p_in=p_in, locality=locality, threads=threads)
    return SparseSimilarity(n, rp, ci, None, float(ci.size))


def generate_citation(n: int, m: int, seed: int, alpha: float = 2.5, gamma: float = 2.0, locality: bool = False,
                      threads: int = 0) -> SparseSimilarity:
    rp, ci = capi.generate_graph(1, n, m, seed, alpha=alpha, gamma=gamma, locality=locality, threads=threads)
    return SparseSimilarity(n, rp, ci, None, float(ci.size))
