"""Similarity construction on the device (fc_build.cu) vs the reference's host
construction (sparse.hpp:66-75 via oracle/_ref), on bench.py's graphs.

Wall-clock per call (host edge list in, host CSR out, resident on the device):
    python scripts/bench_build.py --config C [--reference]
Prints one JSON line per config.  The input edge list is the generator's upper
triangle in random order, so the sort does the real work.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--reference", action="store_true", help="also time oracle/_ref build_similarity once")
    a = ap.parse_args()
    import bench
    from paper_2506_04045_b200 import api, capi
    cfg = bench.CONFIGS[a.config]
    g = bench.make_graph(cfg)
    col_of = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_ptr))
    k = g.col_idx < col_of
    e = np.stack([g.col_idx[k], col_of[k]], 1)
    del col_of, k
    e = e[np.random.default_rng(1).permutation(len(e))]
    ctx = capi.Context(0)
    times = []
    for _ in range(a.reps + 1):
        t0 = time.perf_counter()
        s = api.build_similarity(g.n, e, ctx=ctx)
        times.append(time.perf_counter() - t0)
    same = (s.row_ptr.tobytes() == g.row_ptr.tobytes() and s.col_idx.tobytes() == g.col_idx.tobytes()
            and s.frob_sq == g.frob_sq)
    out = {"config": a.config, "n": g.n, "edges": int(len(e)), "nnz": int(s.nnz), "device_build_s": min(times[1:]),
           "first_call_s": times[0], "identical_to_generator": bool(same)}
    if a.reference:
        from oracle import Reference
        ref = Reference()
        t0 = time.perf_counter()
        h = ref.build_similarity(g.n, e)
        out["reference_build_s"] = time.perf_counter() - t0
        out["reference_threads"] = 1
        del h
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
