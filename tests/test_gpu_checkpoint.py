"""Checkpoint / resume of a solver session (fc_solver_checkpoint / fc_solver_resume,
SURVEY.md 8(f)4): stop a run after k iterations, save it, reload it into a FRESH
context and finish; trace, iterations, reason and membership must equal the
uninterrupted run bit for bit (and the oracle's)."""
import numpy as np
import pytest

from conftest import random_graph
from oracle import FISTA, FISTA_BT, GPA

import paper_2506_04045_b200 as fc
from paper_2506_04045_b200 import capi

pytestmark = pytest.mark.gpu


def _recs(r):
    return [(i, loss, inc) for (i, loss, inc) in r["records"]]


def _same(a, b):
    assert (a["reason"], a["iterations"], a["final_loss"]) == (b["reason"], b["iterations"], b["final_loss"])
    assert _recs(a) == _recs(b)
    assert a["backtracks"] == b["backtracks"] and a["steps"] == b["steps"]
    assert a["membership"].tobytes() == b["membership"].tobytes()


CASES = [
    ("gpa", dict(method=GPA, max_iter=14), 3),
    ("fista", dict(method=FISTA, max_iter=14), 5),
    ("fista_restart_big_step", dict(method=FISTA, max_iter=16, fista_restart=True, step_scale=40.0), 6),
    ("fista_bt", dict(method=FISTA_BT, max_iter=10, step_scale=30.0), 4),
]


@pytest.mark.parametrize("name,kw,stop", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("vshards", [1, 3])
def test_resume_is_bitwise_uninterrupted(tmp_path, oracle, name, kw, stop, vshards):
    kw = dict(kw)
    scale = kw.pop("step_scale", None)
    g = random_graph(7000, 8.0, 77)
    c = 12
    x0 = oracle.init_random(g.n, c, 9)
    if scale:
        kw["step_size"] = scale * oracle.default_step_size(g)
    conf = capi.Context.config(**kw)

    def fresh():
        t = capi.Context(0) if vshards == 1 else capi.Context(0, virtual_shards=vshards)
        t.upload(g)
        return t

    a = fresh()
    try:
        whole = a.solve(x0, conf)
    finally:
        a.close()
    want = oracle.solve(g, x0, **kw)
    assert whole["membership"].tobytes() == want["membership"].tobytes()

    path = tmp_path / "session.fcckpt"
    b = fresh()
    try:
        b.begin(x0, conf)
        b.run(stop)
        b.sync()
        b.checkpoint(str(path))
    finally:
        b.close()
    r = fresh()
    try:
        r.resume(str(path), conf)
        got = r.finish(g.n, c)
    finally:
        r.close()
    _same(got, whole)


def test_resume_rejects_other_similarity_and_bad_files(tmp_path, oracle):
    g = random_graph(3000, 6.0, 5)
    x0 = oracle.init_random(g.n, 8, 1)
    conf = capi.Context.config(method=FISTA, max_iter=6)
    path = tmp_path / "s.fcckpt"
    t = capi.Context(0)
    try:
        t.upload(g)
        t.begin(x0, conf)
        t.run(2)
        t.checkpoint(str(path))
        other = random_graph(3000, 6.0, 6)
        t.upload(other)
        with pytest.raises(fc.InvalidInput, match="similarity"):
            t.resume(str(path), conf)
        bad = tmp_path / "bad.fcckpt"
        bad.write_bytes(b"not a checkpoint at all" * 10)
        with pytest.raises(fc.IoError, match="not a solver checkpoint"):
            t.resume(str(bad), conf)
        t.upload(g)
        cut = tmp_path / "cut.fcckpt"
        cut.write_bytes(path.read_bytes()[: path.stat().st_size // 2])
        with pytest.raises(fc.IoError, match="truncated"):
            t.resume(str(cut), conf)
        with pytest.raises(fc.IoError):
            t.resume(str(tmp_path / "missing.fcckpt"), conf)
        # the intact file still resumes after the failures
        t.resume(str(path), conf)
        t.finish(g.n, 8, want_x=False)
    finally:
        t.close()


def test_reused_context_bt_then_plain_at_new_c(tmp_path, oracle):
    """One context runs a backtracking solve (allocating the line-search buffers), then a
    plain FISTA session at a different C: the checkpoint layout follows the header (no
    stale backtracking blocks), it resumes into a fresh context AND into a context that
    still holds backtracking buffers, and both continuations equal the uninterrupted run.
    A file with trailing bytes is rejected."""
    g = random_graph(6000, 7.0, 31)
    x8, x12 = oracle.init_random(g.n, 8, 2), oracle.init_random(g.n, 12, 3)
    bt = capi.Context.config(method=FISTA_BT, max_iter=5, step_size=30.0 * oracle.default_step_size(g))
    conf = capi.Context.config(method=FISTA, max_iter=12, fista_restart=True)
    want = oracle.solve(g, x12, method=FISTA, max_iter=12, fista_restart=True)
    path = tmp_path / "plain.fcckpt"
    t = capi.Context(0)
    try:
        t.upload(g)
        t.solve(x8, bt)
        t.begin(x12, conf)
        t.run(4)
        t.sync()
        t.checkpoint(str(path))
        t.finish(g.n, 12, want_x=False)
    finally:
        t.close()
    fresh = capi.Context(0)
    try:
        fresh.upload(g)
        fresh.resume(str(path), conf)
        got = fresh.finish(g.n, 12)
    finally:
        fresh.close()
    assert got["membership"].tobytes() == want["membership"].tobytes()
    assert _recs(got) == [tuple(r) for r in want["records"]]
    held = capi.Context(0)
    try:
        held.upload(g)
        held.solve(x12, capi.Context.config(method=FISTA_BT, max_iter=2))   # bt buffers at C = 12
        held.resume(str(path), conf)
        got2 = held.finish(g.n, 12)
        assert got2["membership"].tobytes() == want["membership"].tobytes()
        longer = tmp_path / "long.fcckpt"
        longer.write_bytes(path.read_bytes() + b"\0" * 8)
        with pytest.raises(fc.IoError, match="trailing"):
            held.resume(str(longer), conf)
    finally:
        held.close()


def test_trace_capacity_keeps_terminating_record(oracle):
    """A trace buffer smaller than the run: intermediate records are dropped, the last slot
    holds the terminating record, n_records counts everything produced."""
    g = random_graph(3000, 6.0, 8)
    x0 = oracle.init_random(g.n, 8, 1)
    want = oracle.solve(g, x0, method=GPA, max_iter=9)
    t = capi.Context(0)
    try:
        t.upload(g)
        got = t.solve(x0, capi.Context.config(method=GPA, max_iter=9), trace_cap=4)
    finally:
        t.close()
    assert got["n_records"] == len(want["records"]) == 10
    assert _recs(got)[:3] == [tuple(r) for r in want["records"][:3]]
    assert _recs(got)[3] == tuple(want["records"][-1])
