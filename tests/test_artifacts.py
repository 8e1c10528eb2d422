"""Binary artifacts: membership ("FCMEMB01") and similarity CSR
("FCCSR001") files round-trip bit for bit; malformed files raise IoError.  CPU only."""
import numpy as np
import pytest

from conftest import random_graph

import paper_2506_04045_b200 as fc
from paper_2506_04045_b200.errors import InvalidInput, IoError


def test_membership_binary_roundtrip(tmp_path):
    rng = np.random.default_rng(1)
    x = rng.random((1000, 7))
    x[::3, 2] = 0.0
    x[5, 1] = -0.0
    p = tmp_path / "m.bin"
    fc.write_membership_binary(x, p)
    assert p.stat().st_size == 8 + 16 + x.size * 8
    y = fc.read_membership_binary(p)
    assert y.shape == x.shape and y.tobytes() == x.tobytes()


def test_membership_binary_errors(tmp_path):
    p = tmp_path / "m.bin"
    fc.write_membership_binary(np.ones((10, 3)) / 3, p)
    raw = p.read_bytes()
    (tmp_path / "a").write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(IoError, match="bad magic"):
        fc.read_membership_binary(tmp_path / "a")
    (tmp_path / "b").write_bytes(raw[:-8])
    with pytest.raises(IoError, match="truncated"):
        fc.read_membership_binary(tmp_path / "b")


@pytest.mark.parametrize("weighted", [False, True])
def test_similarity_binary_roundtrip(tmp_path, weighted):
    g = random_graph(3000, 7.0, 4, weighted=weighted)
    p = tmp_path / "s.csr"
    fc.write_similarity_binary(g, p)
    h = fc.read_similarity_binary(p)
    assert h.n == g.n and h.frob_sq == g.frob_sq
    assert h.row_ptr.tobytes() == g.row_ptr.tobytes() and h.col_idx.tobytes() == g.col_idx.tobytes()
    assert (h.values is None) == (g.values is None)
    if g.values is not None:
        assert h.values.tobytes() == g.values.tobytes()


def test_similarity_binary_errors(tmp_path):
    g = random_graph(500, 5.0, 2)
    p = tmp_path / "s.csr"
    fc.write_similarity_binary(g, p)
    raw = bytearray(p.read_bytes())
    (tmp_path / "t").write_bytes(bytes(raw[:-4]))
    with pytest.raises(IoError, match="truncated"):
        fc.read_similarity_binary(tmp_path / "t")
    bad = bytearray(raw)
    bad[8 + 32 + 8 * 501 + 4 * 3: 8 + 32 + 8 * 501 + 4 * 4] = (10**6).to_bytes(4, "little")
    (tmp_path / "r").write_bytes(bytes(bad))
    with pytest.raises(IoError, match="out of range"):
        fc.read_similarity_binary(tmp_path / "r")
    asym = bytearray(raw)   # point entry 1 of row 0 elsewhere: breaks symmetry
    off = 8 + 32 + 8 * 501
    rp = np.frombuffer(bytes(raw[8 + 32: off]), dtype="<i8")
    row = int(np.argmax(np.diff(rp) >= 2))
    k = int(rp[row]) + 1
    cols = np.frombuffer(bytes(raw[off: off + 4 * g.nnz]), dtype="<u4")
    newc = (int(cols[k]) + 1) % g.n
    if k + 1 < rp[row + 1] and newc >= cols[k + 1]:
        newc = int(cols[k]) - 1 if int(cols[k]) - 1 > cols[k - 1] else int(cols[k])
    asym[off + 4 * k: off + 4 * k + 4] = int(newc).to_bytes(4, "little")
    (tmp_path / "y").write_bytes(bytes(asym))
    if newc != int(cols[k]):
        with pytest.raises(InvalidInput, match="symmetric|strictly"):
            fc.read_similarity_binary(tmp_path / "y")


def test_refine_rng_matches_reference_stream():
    """api._SplitMix64 (refine's random combinations) == the rng.hpp stream restated in
    api.splitmix64_stream and the oracle's C splitmix."""
    from paper_2506_04045_b200 import api
    for seed in [0, 1, 99, 2**63 + 5]:
        r = api._SplitMix64(seed)
        got = [r.next() for _ in range(8)]
        want = [int(v) for v in api.splitmix64_stream(seed, 0, 8)]
        assert got == want
    r = api._SplitMix64(7)
    d = r.next_double()
    assert 0.0 <= d < 1.0
