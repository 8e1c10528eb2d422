"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, exports every
symbol include/fuzzyclust_cuda.h declares, refuses to run without a B200 (no
CPU fallback), and its host-only parts (generator, partition planner) behave."""
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import ROOT

from paper_2506_04045_b200 import build as fcbuild
from paper_2506_04045_b200 import capi
import paper_2506_04045_b200 as fc


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "fuzzyclust_cuda.h")).read()
    return sorted(set(re.findall(r"\b(fc_[a-z_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    L = capi.lib()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(capi.SIGNATURES), "ctypes binding must cover exactly the header"


def test_library_is_sm100a_and_links_nccl():
    out = subprocess.run(["cuobjdump", "--list-elf", fcbuild.LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    ldd = subprocess.run(["ldd", fcbuild.LIB], capture_output=True, text=True).stdout
    assert "libnccl" in ldd


def test_no_cpu_fallback():
    import ctypes as C
    L = capi.lib()
    h = C.c_void_p()
    rc = L.fc_create(C.byref(h), 0, 0, 1, None)
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert rc == 3 and not h.value
        with pytest.raises(fc.DeviceError):
            capi.Context(0)
    else:
        L.fc_destroy(h)


def test_generator_deterministic_across_threads():
    for kind in (0, 1):
        a = capi.generate_graph(kind, 20000, 150000, 5, blocks=4, threads=1)
        b = capi.generate_graph(kind, 20000, 150000, 5, blocks=4, threads=7)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        c = capi.generate_graph(kind, 20000, 150000, 6, blocks=4, threads=3)
        assert not np.array_equal(a[1], c[1])


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("locality", [False, True])
def test_generator_builds_a_plus_i(kind, locality):
    n = 30000
    rp, ci = capi.generate_graph(kind, n, 200000, 2, blocks=8, locality=locality)
    g = fc.SparseSimilarity(n, rp, ci)
    g._validate_symmetry()                       # sorted, unique, symmetric
    rows = np.repeat(np.arange(n), np.diff(rp))
    assert np.sum(rows == ci) == n               # diagonal in every row
    assert g.frob_sq == g.nnz                    # all values 1.0
    edges = (g.nnz - n) // 2
    assert 0.8 * 200000 < edges <= 200000 * 1.3


def test_sbm_block_structure():
    n, blocks = 40000, 8
    rp, ci = capi.generate_graph(0, n, 300000, 3, blocks=blocks, p_in=0.9, locality=True)
    rows = np.repeat(np.arange(n), np.diff(rp))
    off = rows != ci
    same = (rows[off] * blocks // n) == (ci[off].astype(np.int64) * blocks // n)
    assert 0.88 < same.mean() < 0.93


def test_citation_power_law_tail():
    n = 200000
    rp, ci = capi.generate_graph(1, n, 20 * n, 4, alpha=2.5, gamma=2.0)
    deg = np.diff(rp) - 1
    assert 30 < deg.mean() < 50                  # ~2 m / n
    assert deg.max() > 50 * deg.mean()           # heavy tail (hubs)


def test_partition_planner():
    rp, _ = capi.generate_graph(1, 100000, 2_000_000, 4, locality=True)
    for world in (1, 2, 3, 4, 8):
        b = capi.plan_partition(rp, world)
        assert b[0] == 0 and b[-1] == 100000 and np.all(np.diff(b.astype(np.int64)) >= 0)
        assert all(int(x) % 1024 == 0 for x in b[1:-1])
        nnz = np.diff(rp[b.astype(np.int64)])
        assert nnz.max() <= rp[-1] / world + 1024 * np.diff(rp).max()
    tiny = np.arange(101, dtype=np.int64)
    b = capi.plan_partition(tiny, 4)
    assert b[0] == 0 and b[-1] == 100


def test_python_mirror_host_parts(oracle):
    assert list(fc.splitmix64_stream(0, 0, 3)) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]
    st = np.uint64(77)
    import ctypes as C
    s = C.c_uint64(77)
    want = [oracle.lib.fco_splitmix_next_double(C.byref(s)) for _ in range(50)] if hasattr(oracle.lib, "fco_splitmix_next_double") else None
    if want is not None:
        oracle.lib.fco_splitmix_next_double.restype = C.c_double
        s = C.c_uint64(77)
        want = [oracle.lib.fco_splitmix_next_double(C.byref(s)) for _ in range(50)]
        assert list(fc.splitmix64_doubles(77, 0, 50)) == want
    x = np.random.default_rng(0).random((23, 3))
    assert np.array_equal(fc.read_membership_csv(fc.write_membership_csv(x)), x)
    with pytest.raises(fc.InvalidInput):
        fc.read_membership_csv("node_id,x_1\n")
    with pytest.raises(fc.InvalidInput):
        fc.read_membership_csv("node_id,x_1,x_2\n0,0.5,0.5\n1,1.0\n")
    tr = fc.SolverTrace(records=[fc.TraceRecord(0, 12.25), fc.TraceRecord(1, 12.25)])
    assert fc.write_trace_csv(tr) == "iteration,loss\n0,12.25\n1,12.25\n"     # cli_test.cpp:104-111
    assert fc.fista_t_next(1.0) == (1 + 5 ** 0.5) / 2


def test_similarity_construction_errors():
    S = fc.SparseSimilarity
    with pytest.raises(fc.InvalidInput, match="not symmetric"):
        S.from_triplets(3, [(0, 1, 1.0)])
    with pytest.raises(fc.InvalidInput, match="duplicate"):
        S.from_triplets(3, [(0, 0, 1.0), (0, 0, 1.0)])
    with pytest.raises(fc.InvalidInput, match="out of range"):
        S.from_triplets(2, [(0, 2, 1.0)])
    with pytest.raises(fc.InvalidInput, match="asymmetric values"):
        S.from_triplets(2, [(0, 1, 1.0), (1, 0, 2.0)])
    with pytest.raises(fc.IoError):
        S.load_coordinates("# nothing\n")
    s = S.load_coordinates("0 0 1\n0 1 0.5\n1 0 0.5\n1 1 1\n")
    assert s.nnz == 4 and s.values is not None and s.frob_sq == 2.5
    seven = S.build_similarity(7, [(0, 1), (1, 2), (1, 3), (2, 3), (3, 4), (3, 5), (4, 5), (5, 6)])
    assert seven.nnz == 23 and seven.frob_sq == 23.0    # graph_test.cpp:139-161
