"""Second-order refinement (secondorder.hpp:343-368) against the
compiled reference: report fields, statuses, witness directions and witness values
bit for bit.  Pair directions are evaluated by fc_refine_pairs (closed forms of the
reference's HVP path); random combinations through the device HVP."""
import numpy as np
import pytest

from conftest import SEVEN_EDGES, random_graph

import paper_2506_04045_b200 as fc
from paper_2506_04045_b200 import capi

pytestmark = pytest.mark.gpu


def _sparse(d):
    return {(int(i), int(k)): float(d[i, k]) for i, k in np.argwhere(d != 0.0)}


def _check(got: "fc.RefinementReport", want: dict):
    assert got.critical == want["critical"]
    assert got.residual == want["residual"]
    assert int(got.status) == want["status"]
    if not got.critical:
        return
    assert got.directions_generated == want["directions_generated"]
    for mine, ref in [(got.condition_a, want["a"]), (got.condition_b, want["b"])]:
        assert int(mine.status) == ref["status"]
        assert mine.directions_tested == ref["tested"]
        assert mine.used_interior_shortcut == ref["interior_shortcut"]
        assert mine.witness_value == ref["value"]
        assert (mine.witness is None) == (ref["witness"] is None)
        if ref["witness"] is not None:
            assert {k: v for k, v in mine.witness.items() if v != 0.0} == _sparse(ref["witness"])
        if ref["base"] is not None:
            assert {k: v for k, v in mine.witness_base.items() if v != 0.0} == _sparse(ref["base"])


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("c", [2, 3, 5])
def test_uniform_saddle(ctx, reference, c):
    s = fc.SparseSimilarity.build_similarity(7, SEVEN_EDGES)
    x = np.full((7, c), 1.0 / c)
    got = fc.refine(x, s, ctx=ctx)
    _check(got, reference.similarity(s).refine(x))
    assert int(got.status) == 1 and got.directions_generated == 7 * c * (c - 1)


def _converged(oracle, g, c, seed):
    from oracle import FISTA
    x0 = oracle.init_random(g.n, c, seed)
    return oracle.solve(g, x0, method=FISTA, max_iter=20000, fista_restart=True)["membership"]


@pytest.mark.parametrize("n,c,seed", [(30, 3, 2), (60, 4, 3), (120, 3, 5)])
@pytest.mark.parametrize("kw", [dict(), dict(eps_critical=1e9, eps_grad_orth=0.05),
                                dict(eps_critical=1e9, eps_grad_orth=0.5, random_directions=10, seed=7),
                                dict(eps_critical=1e9, eps_grad_orth=5.0, random_directions=10, seed=3),
                                dict(eps_critical=1e9, eps_grad_orth=5.0, budget=17)])
def test_refine_matches_reference(ctx, oracle, reference, n, c, seed, kw):
    g = random_graph(n, 4.0, seed)
    x = _converged(oracle, g, c, seed)
    got = fc.refine(x, g, fc.SecondOrderConfig(**kw), ctx=ctx)
    _check(got, reference.similarity(g).refine(x, **kw))


def test_uniform_saddle_with_random_combinations(ctx, reference):
    s = fc.SparseSimilarity.build_similarity(7, SEVEN_EDGES)
    x = np.full((7, 3), 1.0 / 3)
    for kw in [dict(random_directions=9, seed=1), dict(random_directions=9, seed=1, budget=3)]:
        _check(fc.refine(x, s, fc.SecondOrderConfig(**kw), ctx=ctx), reference.similarity(s).refine(x, **kw))


def test_boundary_point_condition_b(ctx, oracle, reference):
    """A point with exact zeros (one-hot rows) exercises condition (b)'s active set."""
    g = random_graph(40, 3.0, 21)
    x = np.zeros((g.n, 3))
    x[np.arange(g.n), np.arange(g.n) % 3] = 1.0
    for kw in [dict(eps_critical=10.0), dict(eps_critical=10.0, eps_grad_orth=10.0),
               dict(eps_critical=10.0, eps_grad_orth=10.0, random_directions=6, seed=3)]:
        got = fc.refine(x, g, fc.SecondOrderConfig(**kw), ctx=ctx)
        _check(got, reference.similarity(g).refine(x, **kw))
