"""Second order on the device: cross_share and the Hessian-vector
product (objective.hpp:61-90, :182-223) bitwise against the oracle restatement
(itself pinned to the compiled reference in tests/test_oracle_second_order.py) and,
when oracle/_ref is present, against the reference directly."""
import numpy as np
import pytest

from conftest import random_graph

import paper_2506_04045_b200 as fc
from paper_2506_04045_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("c", [1, 3, 8, 16, 20, 32, 64, 128])
def test_cross_share_bitwise(ctx, oracle, c):
    n = 2600
    rng = np.random.default_rng(c)
    a = rng.standard_normal((n, c))
    b = rng.random((n, c))
    ctx.upload(random_graph(n, 3.0, 1))
    got = ctx.cross_share(a, b)
    assert got.tobytes() == oracle.cross_share(a, b).tobytes()


@pytest.mark.parametrize("c,weighted,vshards", [(2, False, 1), (8, False, 1), (12, True, 1), (32, False, 1),
                                                (32, False, 3), (40, True, 1), (64, False, 1), (128, False, 1)])
def test_hessian_vector_product_bitwise(oracle, c, weighted, vshards):
    g = random_graph(4100, 7.0, c + 17, weighted=weighted)
    x = oracle.init_random(g.n, c, 3)
    v = np.random.default_rng(c).standard_normal((g.n, c))
    t = capi.Context(0) if vshards == 1 else capi.Context(0, virtual_shards=vshards)
    try:
        t.upload(g)
        got = t.hessian_vector_product(x, v)
    finally:
        t.close()
    want = oracle.hessian_vector_product(x, v, g)
    assert got.tobytes() == want.tobytes()
    assert fc.frob_inner(got, v) == oracle.frob_inner(want, v)


def test_quadratic_form_matches_reference(reference, oracle):
    g = random_graph(3000, 6.0, 8)
    rs = reference.similarity(g)
    x = oracle.init_random(g.n, 6, 2)
    v = np.random.default_rng(4).standard_normal((g.n, 6))
    want_h, want_q = rs.hessian_vector_product(x, v)
    fc.set_default_context(None)
    got_q = fc.quadratic_form(x, v, g)
    got_h = fc.hessian_vector_product(x, v, g)
    assert got_h.tobytes() == want_h.tobytes()
    assert got_q == want_q


def test_pair_direction_quadratic_form(ctx, oracle):
    """check_condition_a's pairwise directions V = e_k - e_l at one node
    (secondorder.hpp:132-137): <H V, V> through the device HVP equals the oracle."""
    g = random_graph(2048, 5.0, 12)
    c = 4
    x = oracle.init_random(g.n, c, 6)
    ctx.upload(g)
    for (i, k, l) in [(0, 0, 1), (77, 3, 2), (2047, 1, 0)]:
        v = np.zeros((g.n, c))
        v[i, k], v[i, l] = 1.0, -1.0
        h = ctx.hessian_vector_product(x, v)
        assert h.tobytes() == oracle.hessian_vector_product(x, v, g).tobytes()
        assert fc.frob_inner(h, v) == oracle.frob_inner(h, v)


def test_shape_errors(ctx):
    g = random_graph(100, 3.0, 1)
    with pytest.raises(fc.InvalidInput, match="shape"):
        fc.hessian_vector_product(np.zeros((100, 3)), np.zeros((100, 4)), g, ctx=ctx)
    with pytest.raises(fc.InvalidInput, match="size"):
        fc.hessian_vector_product(np.zeros((99, 3)), np.zeros((99, 3)), g, ctx=ctx)
    ctx.upload(g)
    with pytest.raises(fc.InvalidInput, match="C=129"):
        ctx.cross_share(np.zeros((100, 129)), np.zeros((100, 129)))
