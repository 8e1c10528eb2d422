"""Edge-list ingest on the device against the compiled reference's
parse_edge_list / largest_connected_component_nodes / two_core_nodes / the CLI's
load_pipeline (tools/fuzzyclust.cpp:62-89): identical node counts, edge lists,
original-id maps and error messages."""
import numpy as np
import pytest

import paper_2506_04045_b200 as fc
from paper_2506_04045_b200 import capi

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


def _random_text(seed, n_ids, m, comps=3, tails=True, big_ids=True):
    """Several components, pendant trees, duplicates, reversed pairs, self-loops,
    comments, blank / CRLF lines, sparse 64-bit ids."""
    rng = np.random.default_rng(seed)
    if big_ids:
        ids = np.unique(rng.integers(-10**12, 10**12, size=2 * n_ids))[:n_ids]
        rng.shuffle(ids)
    else:
        ids = np.arange(n_ids)
    lines = ["# generated", ""]
    part = np.array_split(np.arange(n_ids), comps)
    for p in part:
        if len(p) < 2:
            continue
        k = max(1, int(m * len(p) / n_ids))
        a = rng.choice(p, k)
        b = rng.choice(p, k)
        for x, y in zip(a.tolist(), b.tolist()):
            lines.append(f"{ids[x]} {ids[y]}")
        if tails:                       # a path hanging off the component
            prev = p[0]
            for t in range(min(5, len(p) - 1)):
                nxt = p[-1 - t]
                lines.append(f"{ids[prev]}\t{ids[nxt]}")
                prev = nxt
    lines += [lines[3], " ".join(reversed(lines[4].split())), f"{ids[0]} {ids[0]}", "   # indented comment", "\r"]
    rng.shuffle(lines)
    return ("\n".join(lines) + "\n").replace("\n", "\r\n", 3).encode()


@pytest.mark.parametrize("seed,n,m,comps", [(1, 50, 120, 3), (2, 2000, 6000, 5), (3, 40000, 90000, 1),
                                            (4, 300, 200, 40)])
@pytest.mark.parametrize("stages", [0, 1, 2])
def test_pipeline_matches_reference(ctx, reference, seed, n, m, comps, stages):
    text = _random_text(seed, n, m, comps)
    pn, ln, nn, edges, ids = reference.load_pipeline(text, stages)
    r = ctx.ingest(text, stages)
    assert (r["parsed_nodes"], r["num_nodes"]) == (pn, nn)
    if stages:
        assert r["lcc_nodes"] == ln
    assert r["edges"].tobytes() == edges.astype(np.uint32).tobytes()
    assert r["original_ids"].tobytes() == ids.astype(np.int64).tobytes()


def test_large_multichunk_text(ctx, reference):
    """> 1 MB: parsed by all host threads in newline-aligned chunks."""
    text = _random_text(7, 200_000, 600_000, 4)
    assert len(text) > 4 << 20
    want = reference.load_pipeline(text, 2)
    r = ctx.ingest(text, 2)
    assert (r["parsed_nodes"], r["lcc_nodes"], r["num_nodes"]) == want[:3]
    assert r["edges"].tobytes() == want[3].astype(np.uint32).tobytes()
    assert r["original_ids"].tobytes() == want[4].tobytes()


BAD = [b"0 x\n", b"0 1\n1 2 3\n", b"# only comments\n\n", b"", b"0 1\n2\n", b"1.5 2\n", b"0 1\n+3 -4 #c\n",
       b"99999999999999999999 1\n", b"0 1\n0x10 5\n", b"5 6\n7 8abc\n", b"-9223372036854775808 1\n\n3 4 5\n"]


@pytest.mark.parametrize("text", BAD)
def test_parse_errors_match_reference(ctx, reference, text):
    from oracle import OracleError
    try:
        want = ("ok", reference.load_pipeline(text, 0)[:3])
    except OracleError as e:
        want = ("err", str(e))
    try:
        r = ctx.ingest(text, 0)
        got = ("ok", (r["parsed_nodes"], r["lcc_nodes"], r["num_nodes"]))
    except fc.IoError as e:
        got = ("err", str(e))
    assert got == want


def test_error_in_a_late_chunk_reports_its_line(ctx, reference):
    from oracle import OracleError
    good = "".join(f"{i} {i + 1}\n" for i in range(300_000)).encode()
    text = good + b"12 oops\n" + good
    with pytest.raises(OracleError) as e1:
        reference.load_pipeline(text, 0)
    with pytest.raises(fc.IoError) as e2:
        ctx.ingest(text, 0)
    assert str(e2.value) == str(e1.value)
    assert "line 300001" in str(e2.value)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_graph_node_ops_match_reference(ctx, reference, seed):
    rng = np.random.default_rng(seed)
    n = 5000
    e = rng.integers(0, n, (3000, 2))
    e = np.sort(e[e[:, 0] != e[:, 1]], axis=1)
    e = np.unique(e, axis=0).astype(np.uint32)
    g = fc.Graph(n, e)
    assert np.array_equal(fc.largest_connected_component_nodes(g, ctx), reference.graph_nodes(n, e, 0))
    assert np.array_equal(fc.two_core_nodes(g, ctx), reference.graph_nodes(n, e, 1))


def test_reference_graph_test_cases(ctx):
    """graph_test.cpp known answers."""
    p = fc.parse_edge_list("10 30\n30 20\n# comment\n\n20 10\n", ctx)
    assert p.original_ids.tolist() == [10, 30, 20]
    g = fc.parse_edge_list("0 1\n1 2\n2 0\n1 1\n0 1\n", ctx).graph
    assert g.num_nodes == 3 and g.edges.tolist() == [[0, 1], [0, 2], [1, 2]]
    assert len(fc.parse_edge_list("0 1\n1 0\n2 1\n", ctx).graph.edges) == 2
    tie = fc.Graph(8, np.array([[0, 1], [1, 2], [0, 2], [3, 4], [4, 5], [6, 7]], np.uint32))
    lcc = fc.largest_connected_component(tie, ctx)
    assert lcc.num_nodes == 3 and len(lcc.edges) == 3
    path = fc.Graph(4, np.array([[0, 1], [1, 2], [2, 3]], np.uint32))
    assert fc.prune_degree_one(path, ctx).num_nodes == 0
    cyc = fc.Graph(5, np.array([[0, 1], [1, 2], [0, 2], [2, 3], [3, 4]], np.uint32))
    core = fc.prune_degree_one(cyc, ctx)
    assert core.num_nodes == 3 and fc.prune_degree_one(core, ctx).num_nodes == 3
    with pytest.raises(fc.InvalidInput, match="empty graph"):
        fc.largest_connected_component_nodes(fc.Graph(0, np.zeros((0, 2), np.uint32)), ctx)
    with pytest.raises(fc.InvalidInput, match="empty after preprocessing"):
        fc.load_pipeline("0 1\n1 2\n", prune=True, ctx=ctx)
