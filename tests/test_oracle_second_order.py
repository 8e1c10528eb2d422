"""CPU: the oracle's restatement of cross_share / hessian_vector_product /
quadratic_form (oracle/fc_oracle.c) is bitwise equal to the compiled reference
(objective.hpp:61-90, :182-223 via oracle/_ref)."""
import numpy as np
import pytest

from conftest import random_graph


@pytest.mark.parametrize("c,weighted", [(1, False), (5, False), (9, True), (32, False)])
def test_hvp_restatement_pinned_to_reference(oracle, reference, c, weighted):
    g = random_graph(2200, 6.0, c + 3, weighted=weighted)
    rs = reference.similarity(g)
    x = oracle.init_random(g.n, c, 2)
    v = np.random.default_rng(c).standard_normal((g.n, c))
    want_h, want_q = rs.hessian_vector_product(x, v)
    got_h = oracle.hessian_vector_product(x, v, g)
    assert got_h.tobytes() == want_h.tobytes()
    assert oracle.frob_inner(got_h, v) == want_q
    assert oracle.cross_share(v, x).tobytes() == reference.cross_share(v, x).tobytes()
