"""Drive every kernel variant on small inputs, for compute-sanitizer.

    compute-sanitizer --tool {memcheck,racecheck,initcheck,synccheck} python scripts/sanitize_run.py [--quick]

Variants: default dispatch, FC_SWEEP=tma (TMA gather4 sweep), FC_SWEEP=groups,
FC_STEP=big, FC_GRAPHS=0 (kernel-by-kernel enqueue), FC_HEAVY_DEG=8 (heavy-row
phase of k_sweep / k_sweep_small on every hub), FC_OVERLAP=1 (Gram on a side stream),
virtual shards (ordered combine chain).  Each runs GPA, FISTA with restart and
FISTA with backtracking at C in {1, 3, 8, 16, 32, 48, 64, 128} on a small power-law-ish
graph (a few hubs so the heavy-row path runs), plus the granular operators, the batched
projection, checkpoint/resume, device construction, ingest and the second-order
operators.  Every solve is also compared bitwise with the oracle (a sanity check that
the instrumented run computed the same thing).  Exit code 0 = all equal.
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def graph(n, seed):
    from paper_2506_04045_b200 import SparseSimilarity
    rng = np.random.default_rng(seed)
    m = 4 * n
    u = rng.integers(0, n, m)
    v = np.where(rng.random(m) < 0.3, rng.integers(0, 8, m), rng.integers(0, n, m))   # hubs 0..7
    k = u != v
    e = np.unique(np.sort(np.stack([u[k], v[k]], 1), 1), axis=0)
    return SparseSimilarity.build_similarity(n, e)


def main():
    quick = "--quick" in sys.argv
    from oracle import FISTA, FISTA_BT, GPA, Oracle
    import paper_2506_04045_b200 as fc
    from paper_2506_04045_b200 import capi
    orc = Oracle()
    g = graph(2500, 1)
    cs = (1, 3, 8, 16, 32, 48, 64, 128) if not quick else (3, 16, 32, 64)
    variants = [{}, {"FC_SWEEP": "tma"}, {"FC_SWEEP": "groups"}, {"FC_STEP": "big"}, {"FC_GRAPHS": "0"},
                {"FC_HEAVY_DEG": "8"}, {"FC_OVERLAP": "1"}, {"FC_OVERLAP": "0"}, {"FC_PAIR": "1"},
                {"FC_STEP": "wide1"}, {"FC_FUSE": "1"}, {"_vshards": 3}, {"_tol": 1}]
    if quick:
        variants = [v for v in variants if not v or "FC_HEAVY_DEG" in v or "_vshards" in v or "_tol" in v]
    bad = 0
    tau = orc.default_step_size(g)
    for var in variants:
        env = {k: v for k, v in var.items() if not k.startswith("_")}
        saved = {k: os.environ.get(k) for k in env}
        os.environ.update(env)
        ctx = capi.Context(0, virtual_shards=var["_vshards"]) if "_vshards" in var else capi.Context(0)
        tol = bool(var.get("_tol"))
        try:
            if tol:
                ctx.set_parity_mode(1)
            ctx.upload(g)
            for c in cs:
                if var.get("FC_SWEEP") == "tma" and c % 4:
                    continue
                x0 = orc.init_random(g.n, c, 5)
                for kw in (dict(method=GPA, max_iter=3), dict(method=FISTA, max_iter=4, fista_restart=True,
                                                               step_size=40 * tau),
                           dict(method=FISTA_BT, max_iter=3, step_size=30 * tau)):
                    if tol and (kw["method"] == FISTA_BT or c > 128):
                        continue
                    got = ctx.solve(x0, capi.Context.config(**kw))
                    want = orc.solve(g, x0, **kw)
                    if tol:                                   # north-star bar instead of bitwise
                        ok = (float(np.abs(got["membership"] - want["membership"]).max()) <= 1e-7
                              and all(abs(a[1] - b[1]) <= 1e-9 * abs(b[1])
                                      for a, b in zip(got["records"], want["records"])))
                    else:
                        ok = (got["membership"].tobytes() == want["membership"].tobytes()
                              and [r[:2] for r in got["records"]] == [r[:2] for r in want["records"]])
                    if not ok:
                        bad += 1
                        print("MISMATCH", var, c, kw, flush=True)
                # granular operators
                gm = ctx.share_matrix(x0)
                ctx.fused_column_pass(x0)
                ctx.gpa_step(x0, gm, tau)
                ctx.project_simplex_rows(x0 + 0.1)
            print("variant ok" if not bad else "variant had mismatches", var, flush=True)
        finally:
            ctx.close()
            for k, v in saved.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
    # session checkpoint / resume, device construction, ingest, second order
    ctx = capi.Context(0)
    try:
        ctx.upload(g)
        x0 = orc.init_random(g.n, 8, 2)
        conf = capi.Context.config(method=FISTA, max_iter=6, fista_restart=True)
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "s.fcckpt")
            ctx.begin(x0, conf)
            ctx.run(3)
            ctx.sync()
            ctx.checkpoint(p)
            ctx.finish(g.n, 8, want_x=False)
            ctx.resume(p, conf)
            ctx.finish(g.n, 8)
        col_of = np.repeat(np.arange(g.n, dtype=np.uint32), np.diff(g.row_ptr))
        k = g.col_idx < col_of
        e = np.stack([g.col_idx[k], col_of[k]], 1)[::-1].copy()
        s = fc.build_similarity(g.n, e, ctx=ctx)
        assert s.col_idx.tobytes() == g.col_idx.tobytes()
        text = "".join(f"{a * 7 + 3} {b * 7 + 3}\n" for a, b in e[:4000]).encode()
        fc.load_pipeline(text, ctx=ctx)
        ctx.upload(g)
        v = orc.init_random(g.n, 8, 3) - x0
        fc.hessian_vector_product(x0, v, g, ctx=ctx)
    finally:
        ctx.close()
    print("sanitize_run done, mismatches:", bad, flush=True)
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
