"""GPU parity: the CUDA path (through the C ABI) against the oracle, bitwise.

Bar (BASELINE north_star): objective within 1e-9 relative at every trace
record, U within 1e-7 max-abs, identical support, identical iteration count and
termination reason.  The implementation reproduces the reference's arithmetic
order, so every check here is exact equality (stricter than the bar).
"""
import hashlib

import numpy as np
import pytest

from conftest import load_golden, random_graph
from oracle import FISTA, FISTA_BT, GPA

pytestmark = pytest.mark.gpu

import paper_2506_04045_b200 as fc  # noqa: E402
from paper_2506_04045_b200 import capi  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def recs(r):
    return [(it, float(l).hex(), inc) for it, l, inc in r["records"]]


def assert_same_run(got, want):
    assert (got["reason"], got["iterations"]) == (want["reason"], want["iterations"])
    assert recs(got) == recs(want)
    assert got["final_loss"] == want["final_loss"]
    assert np.array_equal(got["membership"], want["membership"])
    assert np.array_equal(got["membership"] == 0.0, want["membership"] == 0.0)


def cfg(**kw):
    return capi.Context.config(**kw)


# ---- projection ------------------------------------------------------------------------------
def test_projection_fixture_bitwise(ctx):
    for case in load_golden("misc.json")["projections"]:
        x = np.array([float.fromhex(v) for v in case["x"]])
        want = np.array([float.fromhex(v) for v in case["y"]])
        got = ctx.project_simplex_rows(x.reshape(1, -1))[0]
        assert np.array_equal(got, want), len(x)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5, 7, 8, 9, 15, 16, 17, 31, 32, 33, 47, 64, 65, 100, 128, 129, 200, 256])
def test_projection_batch_bitwise(ctx, oracle, c):
    rng = np.random.default_rng(c)
    rows = 3000
    x = rng.normal(0.0, 1.0, size=(rows, c)) * rng.choice([0.01, 1.0, 100.0], size=(rows, 1))
    x[::7] = np.round(x[::7] * 4) / 4          # ties
    x[::11, : max(1, c // 2)] = 0.3            # more ties
    got = ctx.project_simplex_rows(x)
    want = np.stack([oracle.project_simplex(r) for r in x])
    assert np.array_equal(got, want)


def test_projection_known_and_errors(ctx):
    assert list(ctx.project_simplex_rows(np.array([[0.8, 0.8]]))[0]) == [0.5, 0.5]
    assert list(ctx.project_simplex_rows(np.array([[2.0, 0.0]]))[0]) == [1.0, 0.0]
    assert list(ctx.project_simplex_rows(np.array([[-3.7]]))[0]) == [1.0]
    with pytest.raises(fc.InvalidInput, match="non-finite"):
        ctx.project_simplex_rows(np.array([[0.1, np.nan]]))
    with pytest.raises(fc.InvalidInput, match="non-finite"):
        ctx.project_simplex_rows(np.array([[np.inf, 0.0], [0.2, 0.3]]))


def test_init_membership_random_bitwise(ctx, oracle):
    for n, c, seed in [(50, 3, 42), (1000, 8, 1), (777, 33, 5)]:
        x = fc.init_membership(n, c, fc.InitStrategy(fc.InitKind.kRandom, seed), ctx=ctx)
        assert np.array_equal(x, oracle.init_random(n, c, seed))


# ---- granular operators ---------------------------------------------------------------------
@pytest.mark.parametrize("n,c,weighted", [(7, 2, False), (1, 1, False), (1023, 3, False), (1025, 8, True),
                                          (3000, 16, False), (2500, 32, True), (2100, 33, False),
                                          (1500, 64, False), (1200, 100, False), (900, 128, True)])
def test_granular_ops_bitwise(ctx, oracle, n, c, weighted):
    g = random_graph(n, 7.0, n + c, weighted)
    ctx.upload(g)
    x = oracle.init_random(n, c, 3)
    gm = ctx.share_matrix(x)
    assert np.array_equal(gm, oracle.share_matrix(x))
    xs, merge = ctx.fused_column_pass(x)
    xs_o, merge_o = oracle.fused_column_pass(x, g)
    assert np.array_equal(xs, xs_o) and merge == merge_o
    assert ctx.loss_decomposed(x, gm) == oracle.loss_decomposed(x, g, gm)
    tau = oracle.default_step_size(g)
    for step in (tau, 40 * tau, 5000 * tau):
        assert np.array_equal(ctx.gpa_step_fused(x, gm, xs, step), oracle.gpa_step_fused(x, gm, xs_o, step))
        assert np.array_equal(ctx.gpa_step(x, gm, step), oracle.gpa_step_fused(x, gm, xs_o, step))


def test_gpa_step_nonsymmetric_share(ctx, oracle):
    """gpa_step_fused takes any C x C matrix (ShareMatrix::apply reads row k)."""
    g = random_graph(800, 5.0, 3)
    ctx.upload(g)
    x = oracle.init_random(g.n, 5, 1)
    share = np.random.default_rng(0).normal(size=(5, 5)) * 100
    xs, _ = oracle.fused_column_pass(x, g)
    assert np.array_equal(ctx.gpa_step_fused(x, share, xs, 1e-3), oracle.gpa_step_fused(x, share, xs, 1e-3))


def test_zero_similarity_column(ctx, oracle):
    """objective_test.cpp:105-116: node 2 has no entries at all (not even s_22)."""
    s = fc.SparseSimilarity.from_triplets(3, [(0, 0, 1.0), (1, 1, 1.0), (0, 1, 1.0), (1, 0, 1.0)])
    ctx.upload(s)
    x = oracle.init_random(3, 2, 5)
    xs, m = ctx.fused_column_pass(x)
    xs_o, m_o = oracle.fused_column_pass(x, s)
    assert np.array_equal(xs, xs_o) and m == m_o and np.all(xs[2] == 0.0)


# ---- solver: goldens from the real reference ---------------------------------------------------
@pytest.mark.parametrize("run", load_golden("seven_node.json")["runs"], ids=lambda r: r["name"])
def test_seven_node_solver_vs_reference_fixture(ctx, seven, run):
    ctx.upload(seven)
    x0 = np.array(run["x0"])
    kw = dict(run["config"])
    r = ctx.solve(x0, cfg(**kw))
    assert (r["reason"], r["iterations"]) == (run["reason"], run["iterations"])
    assert recs(r) == [tuple(x) for x in run["records"]]
    want = np.array([[float.fromhex(v) for v in row] for row in run["membership"]])
    assert np.array_equal(r["membership"], want)


def test_config_a_vs_reference_fixture(ctx):
    gold = load_golden("config_a.json")
    gg = gold["graph"]
    g = fc.generate_sbm(gg["n"], gg["m"], gg["blocks"], gg["seed"], p_in=gg["p_in"], locality=gg["locality"])
    assert sha(g.col_idx) == gg["col_idx_sha256"]
    ctx.upload(g)
    x0 = fc.init_membership(g.n, 8, fc.InitStrategy(fc.InitKind.kRandom, 1), ctx=ctx)
    assert sha(x0) == gold["x0"]["sha256"]
    for run in gold["runs"]:
        r = ctx.solve(x0, cfg(**run["config"]))
        assert (r["reason"], r["iterations"]) == (run["reason"], run["iterations"]), run["name"]
        assert recs(r) == [tuple(x) for x in run["records"]], run["name"]
        assert sha(r["membership"]) == run["membership_sha256"], run["name"]


# ---- solver vs oracle over a grid of shapes -----------------------------------------------------
@pytest.mark.parametrize("n,c,weighted", [(2, 1, False), (700, 2, False), (1024, 4, True), (2049, 8, False),
                                          (3000, 16, True), (2500, 32, False), (1300, 64, False),
                                          (1000, 128, False)])
@pytest.mark.parametrize("method,restart", [(GPA, False), (FISTA, True), (FISTA, False)])
def test_solver_vs_oracle(ctx, oracle, n, c, weighted, method, restart):
    g = random_graph(n, 8.0, n * 7 + c, weighted)
    ctx.upload(g)
    x0 = oracle.init_random(n, c, c)
    tau = oracle.default_step_size(g)
    for step in (0.0, 30 * tau):
        kw = dict(method=method, step_size=step, max_iter=30, fista_restart=restart)
        assert_same_run(ctx.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))


def test_solver_tol_and_trace_every(ctx, oracle):
    g = random_graph(3000, 6.0, 17)
    ctx.upload(g)
    x0 = oracle.init_random(g.n, 4, 2)
    tau = oracle.default_step_size(g)
    for kw in [dict(method=GPA, step_size=50 * tau, max_iter=500, tol=1e-3, trace_every=7),
               dict(method=FISTA, step_size=50 * tau, max_iter=500, tol=1e-3, trace_every=5),
               dict(method=FISTA, step_size=400 * tau, max_iter=300, trace_every=3),
               dict(method=FISTA, step_size=400 * tau, max_iter=300, fista_restart=True, trace_every=4)]:
        assert_same_run(ctx.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))


def test_solver_input_validation(ctx, seven):
    ctx.upload(seven)
    with pytest.raises(fc.InvalidInput, match="simplex constraint"):
        ctx.solve(np.zeros((7, 2)), cfg(method=GPA))
    with pytest.raises(fc.InvalidInput, match="non-finite entry"):
        x = np.full((7, 2), 0.5)
        x[3, 1] = np.nan
        ctx.solve(x, cfg(method=FISTA))
    with pytest.raises(fc.InvalidInput, match="max_iter"):
        ctx.solve(np.full((7, 2), 0.5), cfg(method=GPA, max_iter=0))
    with pytest.raises(fc.InvalidInput, match="step_size"):
        ctx.solve(np.full((7, 2), 0.5), cfg(method=GPA, step_size=-1.0))


def test_solver_divergence_raises_like_reference(ctx, oracle):
    """A step so large that x - tau*grad overflows: the reference throws
    InvalidInput("project_simplex: non-finite entry") (simplex.hpp:21-23)."""
    from oracle import OracleError
    g = random_graph(500, 6.0, 3)
    ctx.upload(g)
    x0 = oracle.init_random(g.n, 3, 1)
    kw = dict(method=GPA, step_size=1e306, max_iter=5)
    with pytest.raises(OracleError, match="non-finite"):
        oracle.solve(g, x0, **kw)
    with pytest.raises(fc.InvalidInput, match="non-finite"):
        ctx.solve(x0, cfg(**kw))


def test_stateful_session_matches_solve(ctx, oracle):
    g = random_graph(4000, 6.0, 21)
    ctx.upload(g)
    x0 = oracle.init_random(g.n, 8, 4)
    c = cfg(method=FISTA, max_iter=12, fista_restart=True)
    ctx.begin(x0, c)
    ctx.run(5)
    assert not ctx.sync()
    ctx.run(20)                     # extra passes after max_iter are no-ops
    assert ctx.sync()
    r = ctx.end(g.n, 8)
    assert_same_run(r, oracle.solve(g, x0, method=FISTA, max_iter=12, fista_restart=True))


# ---- virtual shards: the multi-GPU partition + ordered chain on one device -------------------
@pytest.mark.parametrize("shards", [2, 3, 8])
def test_virtual_shards_bitwise(oracle, shards):
    v = capi.Context(0, virtual_shards=shards)
    try:
        g = random_graph(9000, 6.0, 5)
        v.upload(g)
        b = v.partition()
        assert b[0] == 0 and b[-1] == g.n and len(b) == shards + 1
        assert all(int(x) % 1024 == 0 for x in b[1:-1])
        x0 = oracle.init_random(g.n, 8, 9)
        for kw in [dict(method=GPA, max_iter=15), dict(method=FISTA, max_iter=15, fista_restart=True)]:
            assert_same_run(v.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
        assert np.array_equal(v.share_matrix(x0), oracle.share_matrix(x0))
        xs, m = v.fused_column_pass(x0)
        xs_o, m_o = oracle.fused_column_pass(x0, g)
        assert np.array_equal(xs, xs_o) and m == m_o
    finally:
        v.close()


# ---- backtracking (parity by restatement; unpinned by the reference) ---------------------------
@pytest.mark.parametrize("c", [3, 8, 12, 16, 32, 40])
def test_backtracking_vs_restatement(ctx, oracle, c):
    """k_step_t's backtracking row terms (C <= 16, exact and padded widths) and the
    lane-parallel k_step (C = 32, 40) against the restatement."""
    g = random_graph(5000, 8.0, 13)
    ctx.upload(g)
    x0 = oracle.init_random(g.n, c, 7)
    tau = oracle.default_step_size(g)
    for kw in [dict(method=FISTA_BT, max_iter=25, fista_restart=True),
               dict(method=FISTA_BT, step_size=5000 * tau, max_iter=40, fista_restart=True, bt_eta=2.0, bt_max=60),
               dict(method=FISTA_BT, step_size=300 * tau, max_iter=40, bt_eta=1.5, bt_max=3)]:
        got = ctx.solve(x0, cfg(**kw))
        want = oracle.solve(g, x0, **kw)
        assert_same_run(got, want)
        assert got["backtracks"] == want["backtracks"] and got["steps"] == want["steps"]


# ---- scale: properties at a size the oracle is too slow for --------------------------------------
def test_large_sbm_properties(ctx):
    g = fc.generate_sbm(400_000, 8_000_000, 16, seed=3)
    ctx.upload(g)
    x0 = fc.init_membership(g.n, 16, fc.InitStrategy(fc.InitKind.kRandom, 1), ctx=ctx)
    r = ctx.solve(x0, cfg(method=FISTA, max_iter=6, fista_restart=True))
    x = r["membership"]
    assert np.all(x >= 0.0) and np.max(np.abs(x.sum(1) - 1.0)) <= 1e-12
    # the final loss equals a fresh evaluation at the returned point
    gm = ctx.share_matrix(x)
    ctx.upload(g)
    assert ctx.loss_decomposed(x, gm) == r["final_loss"]
    # and the device run is deterministic
    r2 = ctx.solve(x0, cfg(method=FISTA, max_iter=6, fista_restart=True))
    assert np.array_equal(r2["membership"], x) and recs(r2) == recs(r)


# ---- the TMA gather4 sweep variant (FC_SWEEP=tma) ------------------------------------------------
@pytest.mark.parametrize("n,c", [(3000, 20), (5000, 32), (2100, 64), (1500, 128)])
def test_tma_sweep_variant_bitwise(oracle, n, c, monkeypatch):
    monkeypatch.setenv("FC_SWEEP", "tma")
    t = capi.Context(0)
    try:
        g = random_graph(n, 9.0, n + c)
        t.upload(g)
        x0 = oracle.init_random(n, c, 2)
        for kw in [dict(method=GPA, max_iter=12), dict(method=FISTA, max_iter=12, fista_restart=True)]:
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
        xs, m = t.fused_column_pass(x0)
        xs_o, m_o = oracle.fused_column_pass(x0, g)
        assert np.array_equal(xs, xs_o) and m == m_o
    finally:
        t.close()


# ---- the NCCL code path on one GPU (1-rank communicator) ------------------------------------
@pytest.mark.parametrize("allgather", ["grouped", "padded"])
def test_nccl_path_single_rank_bitwise(oracle, monkeypatch, allgather):
    """FC_FORCE_NCCL=1 runs the multi-GPU schedule (grouped-broadcast or padded
    ncclAllGather, recv -> combine -> send -> broadcast chain, FISTA + backtracking with
    the per-pass plan read) through a real 1-rank NCCL communicator; results must stay
    bitwise equal to the oracle."""
    monkeypatch.setenv("FC_FORCE_NCCL", "1")
    monkeypatch.setenv("FC_ALLGATHER", allgather)
    t = capi.Context(0, rank=0, world=1, nccl_id=capi.nccl_unique_id())
    try:
        g = random_graph(6000, 7.0, 31)
        t.upload(g)
        x0 = oracle.init_random(g.n, 16, 4)
        for kw in [dict(method=GPA, max_iter=10), dict(method=FISTA, max_iter=10, fista_restart=True),
                   dict(method=FISTA, max_iter=10, step_size=40 * oracle.default_step_size(g)),
                   dict(method=FISTA_BT, max_iter=6, step_size=300 * oracle.default_step_size(g))]:
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
        with pytest.raises(fc.InvalidInput, match="single-rank"):
            t.share_matrix(x0)
    finally:
        t.close()


@pytest.mark.parametrize("n,c", [(900, 40), (700, 200), (600, 256)])
def test_wide_step_odd_and_max_widths(ctx, oracle, n, c):
    g = random_graph(n, 9.0, n + c)
    ctx.upload(g)
    x0 = oracle.init_random(n, c, 8)
    tau = oracle.default_step_size(g)
    for kw in [dict(method=GPA, max_iter=8), dict(method=FISTA, max_iter=8, step_size=50 * tau, fista_restart=True)]:
        assert_same_run(ctx.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))


# ---- heavy-row first phase of k_sweep (power-law hubs scheduled first) -----------------------
@pytest.mark.parametrize("c,vshards", [(32, 1), (20, 1), (64, 1), (32, 3), (8, 1), (3, 2)])
def test_heavy_row_phase_bitwise(oracle, c, vshards, monkeypatch):
    """FC_HEAVY_DEG=24 makes many rows of a small citation graph 'heavy' (processed
    one per warp before the 32-row strips, and skipped by the strips, including
    runs of consecutive heavy rows and heavy first/last rows of a strip)."""
    monkeypatch.setenv("FC_HEAVY_DEG", "24")
    g = fc.generate_citation(30_000, 400_000, seed=3)
    x0 = oracle.init_random(g.n, c, 5)
    t = capi.Context(0) if vshards == 1 else capi.Context(0, virtual_shards=vshards)
    try:
        t.upload(g)
        for kw in [dict(method=GPA, max_iter=6), dict(method=FISTA, max_iter=8, fista_restart=True)]:
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
        if vshards == 1:
            xs, m = t.fused_column_pass(x0)
            xs_o, m_o = oracle.fused_column_pass(x0, g)
            assert np.array_equal(xs, xs_o) and m == m_o
    finally:
        t.close()


# ---- Gram tile shapes of the many-block path (TS = 4, TS = 8 from C = 64) -------------------
@pytest.mark.parametrize("c", [32, 64, 72])
def test_many_block_gram_tiles_bitwise(oracle, c):
    """N = 310k (303 blocks of 1024 rows, more than 2 per SM): k_gram's 4x4 (C < 64) and
    8x8 (C >= 64, C = 72 exercises the padded width) register tiles vs the oracle."""
    g = random_graph(310_000, 5.0, 40 + c)
    x0 = oracle.init_random(g.n, c, 3)
    t = capi.Context(0)
    try:
        t.upload(g)
        kw = dict(method=FISTA, max_iter=2, fista_restart=True)
        assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
        assert t.share_matrix(x0).tobytes() == oracle.share_matrix(x0).tobytes()
    finally:
        t.close()


# ---- live reference at a benchmark size (config B's graph) ------------------------------------
def test_config_b_graph_bitwise_vs_compiled_reference(reference):
    """1e6 nodes / 4.1e7 nonzeros (bench config B): the device solver and the compiled
    reference (all host cores) from the same x0; scripts/parity_at_scale.py does the
    same for configs A, C and E8-E128 (profiles/r01/parity_at_scale.jsonl)."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    g = bench.make_graph(bench.CONFIGS["B"])
    x0_ref = reference.init_membership(g.n, 16, 0, 1, 0)
    t = capi.Context(0)
    try:
        x0 = fc.init_membership(g.n, 16, fc.InitStrategy(fc.InitKind.kRandom, 1), ctx=t)
        assert x0.tobytes() == x0_ref.tobytes()
        t.upload(g)
        got = t.solve(x0, cfg(method=FISTA, max_iter=3, fista_restart=True))
    finally:
        t.close()
    workers = int(reference.lib.fcref_resolve_workers(os.cpu_count() or 1))
    want = reference.similarity(g, fast=True).solve(x0_ref, method=FISTA, max_iter=3, fista_restart=True,
                                                    workers=workers)
    assert [r[:3] for r in got["records"]] == [tuple(r[:3]) for r in want["records"]]
    assert (got["reason"], got["iterations"], got["final_loss"]) == (want["reason"], want["iterations"],
                                                                    want["final_loss"])
    assert got["membership"].tobytes() == want["membership"].tobytes()


# ---- live reference on the benchmark graphs, with a FISTA restart inside the run -------------
@pytest.mark.parametrize("name", ["E32", "C"])
def test_bench_graph_fista_restart_bitwise_vs_compiled_reference(reference, name):
    """Bench configs E32 (4e6 nodes, 1.6e8 nonzeros) and C (1e7 nodes, 4.1e8 nonzeros, k=32):
    6 FISTA iterations with fista_restart=true at a step size large enough that the momentum
    overshoots and the restart branch (solver.hpp:247-249) fires inside the run.  The device
    solver and the compiled reference (all host cores) start from the same x0; every loss
    record, the restart flags, the reason, the iteration count and the membership must be
    identical bit for bit."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    c, iters = bench.CONFIGS[name]["c"], 6
    g = bench.make_graph(bench.CONFIGS[name])
    x0_ref = reference.init_membership(g.n, c, 0, 1, 0)
    sim = reference.similarity(g, fast=True)
    tau = sim.default_step_size()
    t = capi.Context(0)
    try:
        x0 = fc.init_membership(g.n, c, fc.InitStrategy(fc.InitKind.kRandom, 1), ctx=t)
        assert x0.tobytes() == x0_ref.tobytes()
        t.upload(g)
        assert fc.default_step_size(g, g.n) == tau
        # smallest multiple of the default step at which the restart fires within the run
        # (the device run is bitwise the reference's, so the choice is deterministic)
        for mult in (20.0, 100.0, 400.0, 2000.0, 1e4, 1e5):
            got = t.solve(x0, cfg(method=FISTA, step_size=mult * tau, max_iter=iters, fista_restart=True))
            if any(inc for _, _, inc in got["records"]):
                break
        assert any(inc for _, _, inc in got["records"]), "no restart at any probed step size"
    finally:
        t.close()
    workers = int(reference.lib.fcref_resolve_workers(os.cpu_count() or 1))
    want = sim.solve(x0_ref, method=FISTA, step_size=mult * tau, max_iter=iters, fista_restart=True,
                     workers=workers)
    assert want["iterations"] >= 5
    assert [r[:3] for r in got["records"]] == [tuple(r[:3]) for r in want["records"]]
    assert (got["reason"], got["iterations"], got["final_loss"]) == (want["reason"], want["iterations"],
                                                                    want["final_loss"])
    assert got["membership"].tobytes() == want["membership"].tobytes()


def test_upload_rejects_malformed_csr():
    """fc_upload_csr validates the caller's arrays on the device (monotone row_ptr, columns
    < n, strictly ascending per row) instead of faulting later in a gathering kernel; the
    context stays usable afterwards."""
    from paper_2506_04045_b200 import SparseSimilarity
    rp = np.array([0, 2, 4, 6], np.int64)
    good = np.array([0, 1, 0, 1, 1, 2], np.uint32)
    t = capi.Context(0)
    try:
        for col, msg in ((np.array([0, 1, 0, 7, 1, 2], np.uint32), "out of range in row 1"),
                         (np.array([0, 1, 1, 0, 1, 2], np.uint32), "not strictly ascending"),
                         (np.array([0, 1, 0, 1, 2, 2], np.uint32), "not strictly ascending")):
            with pytest.raises(fc.InvalidInput, match=msg):
                t.upload(SparseSimilarity(3, rp, col, None, 6.0))
        with pytest.raises(fc.InvalidInput, match="row_ptr decreases at row 1"):
            t.upload(SparseSimilarity(3, np.array([0, 1, 0, 6], np.int64), good, None, 6.0))
        g = SparseSimilarity(3, rp, good, None, 6.0)
        t.upload(g)
        x0 = np.full((3, 2), 0.5)
        t.solve(x0, cfg(method=GPA, max_iter=2))
    finally:
        t.close()


@pytest.mark.parametrize("c", [1, 3, 5, 8])
@pytest.mark.parametrize("vshards", [1, 3])
def test_pair_layout_sweep_bitwise(oracle, monkeypatch, c, vshards):
    """FC_PAIR=1 (opt-in): the C <= 8 dual sweep gathers interleaved [bar | prev] rows
    (k_pair_pack + k_sweep_small_pair); FISTA with restart and with backtracking stay
    bitwise equal to the oracle (heavy rows included: FC_HEAVY_DEG=16)."""
    monkeypatch.setenv("FC_PAIR", "1")
    monkeypatch.setenv("FC_HEAVY_DEG", "16")
    g = random_graph(9000, 12.0, 60 + c)
    x0 = oracle.init_random(g.n, c, 2)
    t = capi.Context(0) if vshards == 1 else capi.Context(0, virtual_shards=vshards)
    try:
        t.upload(g)
        for kw in (dict(method=FISTA, max_iter=8, fista_restart=True, step_size=40 * oracle.default_step_size(g)),
                   dict(method=FISTA_BT, max_iter=5, step_size=300 * oracle.default_step_size(g))):
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
    finally:
        t.close()


def ragged_graph(n, seed, weighted):
    """Power-law degrees, two hubs, ~5% empty rows (no diagonal either), optional weights."""
    from paper_2506_04045_b200 import SparseSimilarity
    rng = np.random.default_rng(seed)
    deg = np.minimum(rng.zipf(1.8, n), 400)
    u = np.repeat(np.arange(n), deg)
    v = rng.integers(0, n, len(u))
    hubs = np.concatenate([np.full(n // 2, 7), np.full(n // 3, n - 5)])
    u = np.concatenate([u, hubs])
    v = np.concatenate([v, rng.integers(0, n, len(hubs))])
    empty = rng.random(n) < 0.05
    empty[[7, n - 5]] = False
    k = (u != v) & ~empty[u] & ~empty[v]
    e = np.unique(np.sort(np.stack([u[k], v[k]], 1), 1), axis=0)
    ids = np.flatnonzero(~empty)
    w = rng.uniform(0.1, 2.0, len(e)) if weighted else np.ones(len(e))
    d = rng.uniform(0.5, 1.5, len(ids)) if weighted else np.ones(len(ids))
    t = np.concatenate([np.stack([ids, ids, d], 1), np.stack([e[:, 0], e[:, 1], w], 1),
                        np.stack([e[:, 1], e[:, 0], w], 1)])
    return SparseSimilarity.from_triplets(n, t)


@pytest.mark.parametrize("variant", ["FC_ASYNC=3", "FC_ASYNC=4", "FC_ASYNC=6"])
@pytest.mark.parametrize("c", [1, 3, 8])
@pytest.mark.parametrize("weighted", [False, True])
def test_stream_sweep_bitwise(oracle, monkeypatch, variant, c, weighted):
    """FC_PAIR=1 FC_ASYNC=S (k_sweep_async: per-group flat nonzero streams staged through an
    S-stage cp.async ring, warp-uniform) on a ragged graph (power-law degrees, hubs, empty rows), heavy rows through the
    warp-cooperative phase (FC_HEAVY_DEG=64): FISTA with restart and with backtracking
    bitwise equal to the oracle."""
    monkeypatch.setenv("FC_PAIR", "1")
    k, v = variant.split("=")
    monkeypatch.setenv(k, v)
    monkeypatch.setenv("FC_HEAVY_DEG", "64")
    g = ragged_graph(7000, 90 + c, weighted)
    x0 = oracle.init_random(g.n, c, 4)
    t = capi.Context(0)
    try:
        t.upload(g)
        for kw in (dict(method=FISTA, max_iter=8, fista_restart=True, step_size=40 * oracle.default_step_size(g)),
                   dict(method=FISTA_BT, max_iter=5, step_size=300 * oracle.default_step_size(g))):
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
    finally:
        t.close()


@pytest.mark.parametrize("hot_mb", ["0", "0.05", "1000"])
@pytest.mark.parametrize("c", [3, 16, 32])
def test_hot_row_policy_bitwise(oracle, monkeypatch, hot_mb, c):
    """FC_HOT_MB: the L2 evict_last flag (bit 31 of the stored column index) on none, some
    or all columns -- a cache hint only: FISTA with restart and with backtracking stay
    bitwise equal to the oracle, and so do the granular operators on the flagged CSR."""
    monkeypatch.setenv("FC_HOT_MB", hot_mb)
    g = ragged_graph(6000, 130 + c, True)
    x0 = oracle.init_random(g.n, c, 5)
    t = capi.Context(0)
    try:
        t.upload(g)
        for kw in (dict(method=FISTA, max_iter=8, fista_restart=True, step_size=40 * oracle.default_step_size(g)),
                   dict(method=FISTA_BT, max_iter=5, step_size=300 * oracle.default_step_size(g))):
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
    finally:
        t.close()


@pytest.mark.parametrize("variant", ["t2", "t2x", "tx"])
@pytest.mark.parametrize("c", [3, 16, 20, 32])
def test_step_t_variants_bitwise(oracle, monkeypatch, variant, c):
    """FC_STEP=t2 / t2x (two tiles per warp, bar^{n-2} read per thread, 3 CTAs per SM) and
    tx (runtime-C template at C == G): FISTA with restart and GPA bitwise vs the oracle."""
    monkeypatch.setenv("FC_STEP", variant)
    g = random_graph(7000, 9.0, 70 + c)
    x0 = oracle.init_random(g.n, c, 3)
    t = capi.Context(0)
    try:
        t.upload(g)
        for kw in (dict(method=FISTA, max_iter=8, fista_restart=True, step_size=40 * oracle.default_step_size(g)),
                   dict(method=GPA, max_iter=5)):
            assert_same_run(t.solve(x0, cfg(**kw)), oracle.solve(g, x0, **kw))
    finally:
        t.close()
