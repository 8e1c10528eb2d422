"""CPU baseline of the reference solver (oracle/_ref: the unmodified reference headers)
on the bench graphs, with all host threads and with workers = 1 (SURVEY.md 8(d),
BASELINE.md section 3), and on config C with the locality knob on.

    python scripts/cpu_baseline.py [--configs C,Cloc] [--iters 2] [--one-worker-iters 1]

Prints one JSON line per (config, workers).  Graphs come from the host-only generator
build (oracle/_build/libfcgen.so); no CUDA code runs.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C,Cloc")
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--one-worker-iters", type=int, default=1)
    a = ap.parse_args()
    import bench
    from oracle import FISTA, GPA, Reference
    ref = Reference()
    cores = int(ref.lib.fcref_resolve_workers(os.cpu_count() or 1))
    for name in a.configs.split(","):
        cfg = bench.CONFIGS[name]
        t0 = time.perf_counter()
        g = bench.make_graph(cfg, host_only=True)
        gen_s = time.perf_counter() - t0
        sim = ref.similarity(g, fast=True)
        x0 = ref.init_membership(g.n, cfg["c"], 0, bench.X0_SEED, 0)
        method = GPA if cfg["method"] == "gpa" else FISTA
        for workers, iters in ((cores, a.iters), (1, a.one_worker_iters)):
            r = sim.solve(x0, method=method, max_iter=iters, fista_restart=True, workers=workers, want_x=False)
            el = r["elapsed_ms"]
            per_it = (el[-1] - el[0]) / 1e3 / max(1, len(el) - 1)
            print(json.dumps({"config": name, "workload": bench.config_name(name, cfg), "n": g.n, "nnz": g.nnz,
                              "workers": workers, "host_cpus": os.cpu_count(), "iterations": len(el) - 1,
                              "s_per_iter": per_it, "iter_per_s": 1.0 / per_it, "solve_ms": r["solve_ms"],
                              "graph_gen_s": round(gen_s, 1), "kind": "reference (oracle/_ref)"}), flush=True)
        del sim


if __name__ == "__main__":
    main()
