"""Generate tests/golden/*.json from the REAL reference (oracle/_ref/libfcref.so,
built from the unmodified /root/reference headers by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are small JSON files committed to the repo, so the CPU tests and
the GPU box (which has no /root/reference) can pin both the oracle restatement
and the CUDA path against the reference's own outputs.

Graphs: the paper's 7-node instance (support.hpp:25-36, Fig. 1) and
BASELINE config A (SBM n=10k, ~200k edges, k=8) from our counter-based generator
(its CSR is pinned by hash here, and re-validated through the reference's
from_triplets, which checks sorting, duplicates and symmetry).
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import FISTA, GPA, Reference  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

SEVEN_EDGES = [(0, 1), (1, 2), (1, 3), (2, 3), (3, 4), (3, 5), (4, 5), (5, 6)]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def f64hex(v: float) -> str:
    return float(v).hex()


def run_record(sim, x0, **kw):
    r = sim.solve(x0, **kw)
    return {
        "config": kw,
        "reason": r["reason"],
        "iterations": r["iterations"],
        "final_loss": f64hex(r["final_loss"]),
        "step_size": f64hex(r["step_size"]),
        "records": [[it, f64hex(loss), inc] for it, loss, inc in r["records"]],
        "membership_sha256": sha(r["membership"]),
        "zeros": int((r["membership"] == 0.0).sum()),
    }, r


def main() -> None:
    ref = Reference()
    seven = ref.build_similarity(7, SEVEN_EDGES)
    rp, ci, v = seven.export(7)
    out7 = {"edges": SEVEN_EDGES, "row_ptr": rp.tolist(), "col_idx": ci.tolist(), "frob_sq": seven.frob_sq,
            "default_step": f64hex(seven.default_step_size()), "runs": []}
    cases = [
        ("gpa_random_seed1", 0, 1, dict(method=GPA, step_size=0.1)),
        ("gpa_random_seed2", 0, 2, dict(method=GPA, step_size=0.1)),
        ("gpa_random_seed3", 0, 3, dict(method=GPA, step_size=0.1)),
        ("gpa_rowone", 2, 0, dict(method=GPA, step_size=0.1)),
        ("gpa_uniform", 3, 0, dict(method=GPA, step_size=0.1)),
        ("gpa_maxiter5", 0, 9, dict(method=GPA, step_size=1e-4, max_iter=5)),
        ("gpa_thin10", 0, 4, dict(method=GPA, step_size=0.1, trace_every=10)),
        ("fista_seed12", 0, 12, dict(method=FISTA, step_size=0.05, max_iter=5000)),
        ("fista_plain_seed3", 0, 3, dict(method=FISTA, step_size=0.12, max_iter=2000)),
        ("fista_restart_seed3", 0, 3, dict(method=FISTA, step_size=0.12, max_iter=2000, fista_restart=True)),
        ("fista_auto", 0, 5, dict(method=FISTA, max_iter=300)),
    ]
    for name, kind, seed, kw in cases:
        x0 = ref.init_membership(7, 2, kind, seed, 0)
        rec, r = run_record(seven, x0, **kw)
        rec.update(name=name, init_kind=kind, init_seed=seed, x0=x0.tolist(),
                   membership=[[f64hex(e) for e in row] for row in r["membership"]])
        out7["runs"].append(rec)
    with open(os.path.join(OUT, "seven_node.json"), "w") as f:
        json.dump(out7, f, indent=1)

    # ---- config A --------------------------------------------------------------
    import paper_2506_04045_b200 as fc  # generator only (host code of the library)
    g = fc.generate_sbm(10000, 200000, 8, seed=1)
    sim = ref.similarity(g, fast=False)        # reference from_triplets: validates our CSR
    rp2, ci2, _ = sim.export(g.n)
    assert np.array_equal(rp2, g.row_ptr) and np.array_equal(ci2, g.col_idx)
    x0 = ref.init_membership(g.n, 8, 0, 1, 0)
    tau = sim.default_step_size()
    outA = {"graph": {"kind": "sbm", "n": 10000, "m": 200000, "blocks": 8, "seed": 1, "p_in": 0.9,
                      "locality": False, "nnz": g.nnz, "row_ptr_sha256": sha(g.row_ptr),
                      "col_idx_sha256": sha(g.col_idx)},
            "x0": {"kind": "random", "seed": 1, "c": 8, "sha256": sha(x0)},
            "default_step": f64hex(tau), "runs": []}
    for name, kw in [
        ("gpa_auto_100", dict(method=GPA, max_iter=100)),
        ("gpa_20x_100", dict(method=GPA, max_iter=100, step_size=20 * tau)),
        ("fista_auto_60", dict(method=FISTA, max_iter=60, fista_restart=True)),
        ("fista_20x_60", dict(method=FISTA, max_iter=60, step_size=20 * tau, fista_restart=True)),
        ("fista_20x_norestart", dict(method=FISTA, max_iter=60, step_size=20 * tau)),
    ]:
        rec, _ = run_record(sim, x0, **kw)
        rec["name"] = name
        outA["runs"].append(rec)
    with open(os.path.join(OUT, "config_a.json"), "w") as f:
        json.dump(outA, f, indent=1)

    # ---- splitmix stream + projections -----------------------------------------
    misc = {"splitmix_seed0": [hex(ref.splitmix(0, k)) for k in range(8)],
            "splitmix_seed1234567": [hex(ref.splitmix(1234567, k)) for k in range(8)],
            "projections": []}
    rng = np.random.default_rng(5)
    for c in [1, 2, 3, 4, 7, 8, 16, 31, 32, 33, 64, 100, 128]:
        for scale in (0.5, 3.0, 50.0):
            x = rng.uniform(-scale, scale, size=c)
            y = ref.project_simplex(x)
            misc["projections"].append({"x": [f64hex(e) for e in x], "y": [f64hex(e) for e in y]})
    with open(os.path.join(OUT, "misc.json"), "w") as f:
        json.dump(misc, f, indent=1)
    print("wrote", os.listdir(OUT))


if __name__ == "__main__":
    main()
