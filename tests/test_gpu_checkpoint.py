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
