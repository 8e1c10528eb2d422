"""Edge-list ingest (parse -> LCC -> 2-core) on the device vs the reference's
load_pipeline (oracle/_ref, single thread), on a text edge list made from a bench
graph with random 40-bit node ids.

    python scripts/bench_ingest.py --config B [--reference]
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
    ap.add_argument("--config", default="B")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--reference", action="store_true")
    a = ap.parse_args()
    import bench
    from paper_2506_04045_b200 import capi
    g = bench.make_graph(bench.CONFIGS[a.config])
    col_of = np.repeat(np.arange(g.n, dtype=np.int64), np.diff(g.row_ptr))
    k = g.col_idx.astype(np.int64) < col_of
    e = np.stack([g.col_idx[k].astype(np.int64), col_of[k]], 1)
    rng = np.random.default_rng(3)
    e = e[rng.permutation(len(e))]
    ids = rng.integers(0, 1 << 40, size=g.n)
    t0 = time.perf_counter()
    text = "\n".join(f"{u} {v}" for u, v in zip(ids[e[:, 0]].tolist(), ids[e[:, 1]].tolist())).encode() + b"\n"
    gen_s = time.perf_counter() - t0
    ctx = capi.Context(0)
    times = []
    for _ in range(a.reps + 1):
        t0 = time.perf_counter()
        r = ctx.ingest(text, 2)
        times.append(time.perf_counter() - t0)
    out = {"config": a.config, "text_mb": round(len(text) / 1e6, 1), "edges": int(len(e)),
           "parsed_nodes": r["parsed_nodes"], "lcc_nodes": r["lcc_nodes"], "core_nodes": r["num_nodes"],
           "device_ingest_s": min(times[1:]), "first_call_s": times[0], "text_gen_s": round(gen_s, 1),
           "host_threads": os.cpu_count()}
    if a.reference:
        from oracle import Reference
        t0 = time.perf_counter()
        want = Reference().load_pipeline(text, 2)
        out["reference_s"] = time.perf_counter() - t0
        out["identical"] = bool(want[2] == r["num_nodes"] and want[3].astype(np.uint32).tobytes() == r["edges"].tobytes()
                                and want[4].tobytes() == r["original_ids"].tobytes())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
