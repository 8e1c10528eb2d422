"""GPU construction of the similarity (csrc/fc_build.cu) against the
COMPILED REFERENCE (oracle/_ref: SparseSimilarity::from_triplets / build_similarity,
sparse.hpp:28-75, validate_symmetry :115-139) and the host restatement in
similarity.py: identical CSR arrays and frob_sq bit for bit, the same exception and
message for the first failing entry, and the built matrix resident for the solver
without another upload."""
import numpy as np
import pytest

from conftest import SEVEN_EDGES, random_graph

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2506_04045_b200 import capi
    c = capi.Context(0)
    yield c
    c.close()


def _same(a, b):
    assert a.n == b.n and a.nnz == b.nnz
    assert a.row_ptr.tobytes() == b.row_ptr.tobytes()
    assert a.col_idx.tobytes() == b.col_idx.tobytes()
    assert (a.values is None) == (b.values is None)
    if a.values is not None:
        assert a.values.tobytes() == b.values.tobytes()
    assert a.frob_sq == b.frob_sq


def _weighted_triplets(n, seed, deg=6.0):
    g = random_graph(n, deg, seed, weighted=True)
    col_of = np.repeat(np.arange(n), np.diff(g.row_ptr))
    t = np.stack([g.col_idx.astype(np.float64), col_of.astype(np.float64), g.values], 1)
    rng = np.random.default_rng(seed + 1)
    return g, t[rng.permutation(len(t))]


def test_seven_node_build_similarity(ctx):
    from paper_2506_04045_b200 import SparseSimilarity, api
    want = SparseSimilarity.build_similarity(7, SEVEN_EDGES)
    got = api.build_similarity(7, SEVEN_EDGES, ctx=ctx)
    _same(got, want)
    assert got.frob_sq == 23.0


@pytest.mark.parametrize("n,deg,seed", [(1, 0.0, 1), (100, 3.0, 2), (5000, 8.0, 3), (70000, 12.0, 4)])
def test_build_similarity_matches_host(ctx, n, deg, seed):
    from paper_2506_04045_b200 import SparseSimilarity, api
    rng = np.random.default_rng(seed)
    m = int(n * deg / 2)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    k = u != v
    e = np.unique(np.sort(np.stack([u[k], v[k]], 1), 1), axis=0) if k.any() else np.zeros((0, 2), np.int64)
    e = e[rng.permutation(len(e))]
    want = SparseSimilarity.build_similarity(n, e)
    got = api.build_similarity(n, e, ctx=ctx)
    _same(got, want)


@pytest.mark.parametrize("n,seed", [(50, 5), (3000, 6), (40000, 7)])
def test_from_triplets_weighted_matches_host(ctx, n, seed):
    from paper_2506_04045_b200 import SparseSimilarity, api
    g, t = _weighted_triplets(n, seed)
    want = SparseSimilarity.from_triplets(n, t)
    got = api.from_triplets(n, t, ctx=ctx)
    _same(got, want)
    _same(got, g)


def test_from_triplets_all_ones_is_pattern(ctx):
    from paper_2506_04045_b200 import SparseSimilarity, api
    g = random_graph(2000, 5.0, 9)
    col_of = np.repeat(np.arange(g.n), np.diff(g.row_ptr))
    t = np.stack([g.col_idx, col_of, np.ones(g.nnz)], 1)[::-1]
    got = api.from_triplets(g.n, t, ctx=ctx)
    assert got.values is None and got.frob_sq == float(g.nnz)
    _same(got, SparseSimilarity.from_triplets(g.n, t))


def _host_error(n, t):
    from paper_2506_04045_b200 import SparseSimilarity
    from paper_2506_04045_b200.errors import InvalidInput
    with pytest.raises(InvalidInput) as e:
        SparseSimilarity.from_triplets(n, t)
    return str(e.value)


@pytest.mark.parametrize("case", ["range", "neg", "value", "nan", "value_before_range", "range_before_value",
                                  "dup", "asym_pattern", "asym_value", "asym_value_first"])
def test_from_triplets_errors_match_host(ctx, case):
    from paper_2506_04045_b200 import api
    from paper_2506_04045_b200.errors import InvalidInput
    n = 6
    base = [(0, 0, 1.0), (1, 2, 0.5), (2, 1, 0.5), (3, 4, 2.0), (4, 3, 2.0), (5, 5, 1.0)]
    t = [list(x) for x in base]
    if case == "range":
        t[3][0] = 6
    elif case == "neg":
        t[2][1] = -1
    elif case == "value":
        t[4][2] = -2.0
    elif case == "nan":
        t[1][2] = float("nan")
    elif case == "value_before_range":
        t[1][2] = float("inf")
        t[4][0] = 9
    elif case == "range_before_value":
        t[1][0] = 7
        t[4][2] = -1.0
    elif case == "dup":
        t.append([3, 4, 2.0])
    elif case == "asym_pattern":
        t.append([0, 5, 1.0])
    elif case == "asym_value":
        t[4][2] = 3.0
    elif case == "asym_value_first":
        t[2][2] = 0.25          # (2,1) vs (1,2): column 1 comes first -> "(2, 1)"
        t[3][2] = 1.5
    want = _host_error(n, t)
    with pytest.raises(InvalidInput) as e:
        api.from_triplets(n, t, ctx=ctx)
    assert str(e.value) == want


def test_build_similarity_error_edge_out_of_range(ctx):
    from paper_2506_04045_b200 import SparseSimilarity, api
    from paper_2506_04045_b200.errors import InvalidInput
    with pytest.raises(InvalidInput) as h:
        SparseSimilarity.build_similarity(5, [(0, 1), (2, 5)])
    with pytest.raises(InvalidInput) as d:
        api.build_similarity(5, [(0, 1), (2, 5)], ctx=ctx)
    assert str(d.value) == str(h.value) == "similarity: index out of range"
    with pytest.raises(InvalidInput) as d2:
        api.build_similarity(5, [(0, 1), (1, 0)], ctx=ctx)
    assert str(d2.value) == "similarity: duplicate coordinate entry"


def test_built_similarity_is_resident_and_solves_identically(ctx):
    """Solve right after the device build (no upload) == solve after a host upload."""
    from paper_2506_04045_b200 import api
    from paper_2506_04045_b200.api import Method, SolverConfig
    g0 = random_graph(4000, 7.0, 11)
    col_of = np.repeat(np.arange(g0.n), np.diff(g0.row_ptr))
    k = g0.col_idx < col_of
    e = np.stack([g0.col_idx[k], col_of[k]], 1)
    x0 = api.init_membership(g0.n, 6, ctx=ctx)
    s = api.build_similarity(g0.n, e, ctx=ctx)
    cfg = SolverConfig(method=Method.kFista, max_iter=15)
    r1 = api.solve(x0, s, cfg, ctx=ctx)
    ctx.upload(g0)
    r2 = api.solve(x0, g0, cfg, ctx=ctx)
    assert r1.membership.tobytes() == r2.membership.tobytes()
    assert [r.loss for r in r1.trace.records] == [r.loss for r in r2.trace.records]


def test_build_matches_generator_csr_large(ctx):
    """SBM graph from the CSR generator (1e6 nodes, ~2e7 entries): rebuilding it from its
    shuffled edge list on the device reproduces the generator's CSR exactly."""
    from paper_2506_04045_b200 import api
    g = api.generate_sbm(1_000_000, 10_000_000, 64, seed=5)
    col_of = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_ptr))
    k = g.col_idx < col_of
    e = np.stack([g.col_idx[k], col_of[k]], 1)
    e = e[np.random.default_rng(1).permutation(len(e))]
    got = api.build_similarity(g.n, e, ctx=ctx)
    _same(got, g)


# ---- against the compiled reference (oracle/_ref) -------------------------------------------
def _ref_same(got, ref_sim, n):
    rp, ci, v = ref_sim.export(n)
    assert got.n == n and got.nnz == ci.size
    assert got.row_ptr.tobytes() == rp.tobytes()
    assert got.col_idx.tobytes() == ci.tobytes()
    gv = np.ones(got.nnz) if got.values is None else got.values
    assert gv.tobytes() == v.tobytes()
    assert got.frob_sq == ref_sim.frob_sq


def _ref_error(reference, n, t):
    from oracle import OracleError
    t = np.asarray(t, dtype=np.float64).reshape(-1, 3)
    idx = lambda a: np.where((a < 0) | (a > 0xFFFFFFFF) | ~np.isfinite(a), 0xFFFFFFFF, a).astype(np.uint32)
    with pytest.raises(OracleError) as e:
        reference.from_triplets(n, idx(t[:, 0]), idx(t[:, 1]), t[:, 2])
    assert e.value.code == 2
    return str(e.value)


@pytest.mark.parametrize("n,seed", [(1, 1), (50, 5), (3000, 6), (40000, 7), (300000, 8)])
def test_from_triplets_shuffled_weighted_matches_reference(ctx, reference, n, seed):
    from paper_2506_04045_b200 import api
    _, t = _weighted_triplets(n, seed)
    got = api.from_triplets(n, t, ctx=ctx)
    want = reference.from_triplets(n, t[:, 0].astype(np.uint32), t[:, 1].astype(np.uint32), t[:, 2])
    _ref_same(got, want, n)


@pytest.mark.parametrize("n,deg,seed", [(7, 0.0, 0), (100, 3.0, 2), (5000, 8.0, 3), (200000, 12.0, 4)])
def test_build_similarity_shuffled_matches_reference(ctx, reference, n, deg, seed):
    from paper_2506_04045_b200 import api
    rng = np.random.default_rng(seed)
    m = int(n * deg / 2)
    u, v = rng.integers(0, n, m), rng.integers(0, n, m)
    k = u != v
    e = np.unique(np.sort(np.stack([u[k], v[k]], 1), 1), axis=0) if k.any() else np.zeros((0, 2), np.int64)
    e = e[rng.permutation(len(e))]
    flip = rng.random(len(e)) < 0.5
    e[flip] = e[flip][:, ::-1]                       # either orientation, as an edge list has it
    got = api.build_similarity(n, e, ctx=ctx)
    _ref_same(got, reference.build_similarity(n, e), n)


def test_build_config_b_graph_matches_reference(ctx, reference):
    """Config B's 2.0e7 edges (1e6 nodes), shuffled: the device build equals the reference's
    build_similarity (sort + duplicate check + validate_symmetry) entry for entry."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    from paper_2506_04045_b200 import api
    g = bench.make_graph(bench.CONFIGS["B"])
    col_of = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_ptr))
    k = g.col_idx < col_of
    e = np.stack([g.col_idx[k], col_of[k]], 1)
    e = e[np.random.default_rng(3).permutation(len(e))]
    got = api.build_similarity(g.n, e, ctx=ctx)
    _ref_same(got, reference.build_similarity(g.n, e), g.n)
    _same(got, g)


@pytest.mark.parametrize("case", ["range", "neg", "value", "nan", "value_before_range", "range_before_value",
                                  "dup", "asym_pattern", "asym_value", "asym_value_first", "dup_shuffled"])
def test_from_triplets_errors_match_reference(ctx, reference, case):
    from paper_2506_04045_b200 import api
    from paper_2506_04045_b200.errors import InvalidInput
    n = 6
    base = [(0, 0, 1.0), (1, 2, 0.5), (2, 1, 0.5), (3, 4, 2.0), (4, 3, 2.0), (5, 5, 1.0)]
    t = [list(x) for x in base]
    if case == "range":
        t[3][0] = 6
    elif case == "neg":
        t[2][1] = -1
    elif case == "value":
        t[4][2] = -2.0
    elif case == "nan":
        t[1][2] = float("nan")
    elif case == "value_before_range":
        t[1][2] = float("inf")
        t[4][0] = 9
    elif case == "range_before_value":
        t[1][0] = 7
        t[4][2] = -1.0
    elif case == "dup":
        t.append([3, 4, 2.0])
    elif case == "dup_shuffled":
        t.insert(0, [4, 3, 2.0])
    elif case == "asym_pattern":
        t.append([0, 5, 1.0])
    elif case == "asym_value":
        t[4][2] = 3.0
    elif case == "asym_value_first":
        t[2][2] = 0.25
        t[3][2] = 1.5
    want = _ref_error(reference, n, t)
    with pytest.raises(InvalidInput) as e:
        api.from_triplets(n, t, ctx=ctx)
    assert str(e.value) == want
