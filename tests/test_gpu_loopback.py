"""Multi-rank solver on one GPU through the in-process loopback transport
(fc_loopback: W rank contexts, one host thread each, exchanging through stream-ordered
device copies instead of NCCL).  The ranks run exactly the multi-rank code path of a
one-process-per-GPU run: nnz-balanced 1024-row shards, the allgather of each rank's
new rows, the ordered recv -> combine -> send chain of the block partials and the
broadcast from the last rank (parallel.hpp:36-68 decomposition).
Every rank's result must equal the oracle bit for bit, for GPA, FISTA with restart and
FISTA with backtracking (whose rejected trials need every rank to agree on the replica
each pass writes)."""
import threading

import numpy as np
import pytest

from conftest import random_graph
from oracle import FISTA, FISTA_BT, GPA

from paper_2506_04045_b200 import capi

pytestmark = pytest.mark.gpu


def run_ranks(world, g, x0, conf):
    group = capi.LoopbackGroup(world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            ctx = group.context(r)
            try:
                ctx.upload(g)
                out[r] = (ctx.partition(), ctx.solve(x0, conf))
            finally:
                ctx.close()
        except Exception as e:          # surfaced below (a failing rank must not hang the others)
            errs.append((r, repr(e)))

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    group.close()
    assert not errs, errs
    return out


def same(got, want):
    assert (got["reason"], got["iterations"]) == (want["reason"], want["iterations"])
    assert [r[:3] for r in got["records"]] == [tuple(r[:3]) for r in want["records"]]
    assert got["membership"].tobytes() == want["membership"].tobytes()


CASES = [
    ("gpa", dict(method=GPA, max_iter=6)),
    ("fista_restart", dict(method=FISTA, max_iter=8, fista_restart=True, step_scale=40.0)),
    ("fista_bt", dict(method=FISTA_BT, max_iter=6, step_scale=30.0)),
]


@pytest.mark.parametrize("world", [2, 3, 8])
@pytest.mark.parametrize("c", [8, 32, 48])
@pytest.mark.parametrize("name,kw", CASES, ids=[c[0] for c in CASES])
def test_loopback_ranks_bitwise(oracle, world, c, name, kw):
    g = random_graph(21_000, 9.0, 100 + c)
    x0 = oracle.init_random(g.n, c, 4)
    kw = dict(kw)
    scale = kw.pop("step_scale", None)
    if scale:
        kw["step_size"] = scale * oracle.default_step_size(g)
    want = oracle.solve(g, x0, **kw)
    if name == "fista_bt":
        # grow the initial step until the oracle's line search rejects a trial
        while not any(b > 0 for b in want["backtracks"]) and kw["step_size"] < 1e6:
            kw["step_size"] *= 10.0
            want = oracle.solve(g, x0, **kw)
    res = run_ranks(world, g, x0, capi.Context.config(**kw))
    bounds = res[0][0]
    assert len(bounds) == world + 1 and bounds[-1] == g.n and all(int(b) % 1024 == 0 for b in bounds[:-1])
    for _, got in res:
        same(got, want)
    if name == "fista_bt":
        assert any(b > 0 for b in res[0][1]["backtracks"]), "no rejected line-search trial exercised"


@pytest.mark.parametrize("world", [3, 4])
def test_loopback_empty_shards(oracle, world):
    """n < 1024 * world: some ranks own no rows (and no blocks) but still take part in
    every collective and hold the full replica."""
    g = random_graph(1500, 6.0, 9)
    x0 = oracle.init_random(g.n, 6, 2)
    kw = dict(method=FISTA, max_iter=5, fista_restart=True)
    want = oracle.solve(g, x0, **kw)
    res = run_ranks(world, g, x0, capi.Context.config(**kw))
    assert int(res[0][0][1]) - int(res[0][0][0]) in (0, 1024, 1500)
    for _, got in res:
        same(got, want)


# ---- halo exchange (locality graphs): only the rows other shards reference move ------------
def run_ranks_env(world, g, x0, conf, env):
    import os
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    group = capi.LoopbackGroup(world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            ctx = group.context(r)
            try:
                ctx.upload(g)
                out[r] = (ctx.halo_info(), ctx.solve(x0, conf))
            finally:
                ctx.close()
        except Exception as e:
            errs.append((r, repr(e)))

    try:
        th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=600)
    finally:
        group.close()
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert not errs, errs
    return out


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("method", [GPA, FISTA])
def test_halo_exchange_locality_graph_bitwise(oracle, world, method):
    """Block model with contiguous blocks (locality=1): 90% of the edges stay inside a
    block, so a shard references few rows of the others; the automatic plan picks the
    halo exchange, and every rank's result equals the oracle."""
    import paper_2506_04045_b200 as fc
    g = fc.generate_sbm(64_000, 128_000, 16, seed=3, p_in=0.97, locality=True)
    x0 = oracle.init_random(g.n, 16, 5)
    kw = dict(method=method, max_iter=6, fista_restart=True)
    want = oracle.solve(g, x0, **kw)
    res = run_ranks_env(world, g, x0, capi.Context.config(**kw), {})
    for (mode, recv, _), got in res:
        assert mode == 1 and recv < g.n // 2
        same(got, want)


def test_halo_exchange_forced_on_random_graph(oracle):
    g = random_graph(12_000, 7.0, 77)
    x0 = oracle.init_random(g.n, 8, 6)
    kw = dict(method=FISTA, max_iter=5, fista_restart=True, step_size=40 * oracle.default_step_size(g))
    want = oracle.solve(g, x0, **kw)
    res = run_ranks_env(3, g, x0, capi.Context.config(**kw), {"FC_HALO": "1"})
    for (mode, _, _), got in res:
        assert mode == 1
        same(got, want)
    res = run_ranks_env(3, g, x0, capi.Context.config(**kw), {"FC_HALO": "0"})
    for (mode, _, _), got in res:
        assert mode == 0
        same(got, want)
