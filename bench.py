#!/usr/bin/env python
"""Benchmark: FISTA iterations/s (and edges/s, GB/s vs the HBM roofline) of the
B200 solver on BASELINE configurations, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1: NCCL row-sharded solver)

One "step" = one FISTA iteration (BASELINE metric) over the whole graph.
Workload (default): BASELINE config C -- power-law citation-like graph,
n = 10M nodes, 200M undirected edge draws, k = 32, FISTA, row-partitioned
across the N GPUs (strong scaling: the graph is fixed as N grows).
Inputs (CSR 1.7 GB, U 2.6 GB per replica) are far larger than the 126 MB L2,
so no explicit flush is needed between timed iterations.

--impl reference times the UNMODIFIED reference CPU solver (oracle/_ref, built
from /root/reference headers) on the same graph and metric, with all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (kind, n, m, C, method, extra)
    # m = edge draws, sized so the undirected edge count after merging duplicates and
    # self-loops reaches the BASELINE figure (A: 200,082; B: 20,004,748; C: 200,036,749;
    # E: 80,110,906 edges)
    "A": dict(kind="sbm", n=10_000, m=202_800, c=8, blocks=8, method="gpa"),
    "B": dict(kind="sbm", n=1_000_000, m=20_010_000, c=16, blocks=16, method="fista_bt"),
    "C": dict(kind="citation", n=10_000_000, m=206_100_000, c=32, method="fista"),
    # config C with the locality knob on (ids in citation time order: neighbours near in id
    # space -- L2-friendly gathers on one GPU, halo exchange instead of allgather on N GPUs)
    "Cloc": dict(kind="citation", n=10_000_000, m=206_100_000, c=32, method="fista", locality=True),
    "D": dict(kind="citation", n=70_000_000, m=1_032_000_000, c=32, method="fista"),
    "E8": dict(kind="citation", n=4_000_000, m=82_500_000, c=8, method="fista"),
    "E32": dict(kind="citation", n=4_000_000, m=82_500_000, c=32, method="fista"),
    "E64": dict(kind="citation", n=4_000_000, m=82_500_000, c=64, method="fista"),
    "E128": dict(kind="citation", n=4_000_000, m=82_500_000, c=128, method="fista"),
}
GRAPH_SEED = 1
X0_SEED = 1


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def make_graph(cfg, threads=0, host_only=False):
    """The config's synthetic graph.  host_only: the same generator built without CUDA
    (oracle/_build/libfcgen.so) -- the reference arm must not load the repo's CUDA library."""
    if host_only:
        from oracle import generate_graph
        kind = 0 if cfg["kind"] == "sbm" else 1
        return generate_graph(kind, cfg["n"], cfg["m"], GRAPH_SEED, blocks=cfg.get("blocks", 16), p_in=0.9,
                              alpha=2.5, gamma=2.0, locality=cfg.get("locality", False), threads=threads)
    import paper_2506_04045_b200 as fc
    if cfg["kind"] == "sbm":
        return fc.generate_sbm(cfg["n"], cfg["m"], cfg["blocks"], seed=GRAPH_SEED, p_in=0.9,
                               locality=cfg.get("locality", False), threads=threads)
    return fc.generate_citation(cfg["n"], cfg["m"], seed=GRAPH_SEED, alpha=2.5, gamma=2.0,
                                locality=cfg.get("locality", False), threads=threads)


def shared_graph(cfg, name, rank, world):
    """N > 1: rank 0 generates the graph once and writes it as an FCCSR001 file in
    /dev/shm; every rank maps that file (zero-copy, one page-cache copy for the node)
    instead of each rank regenerating the whole graph in host memory."""
    import paper_2506_04045_b200 as fc
    need = 8 * (cfg["n"] + 1) + 4 * (2 * cfg["m"] + cfg["n"]) + (1 << 26)   # upper bound of the file
    root = "/tmp"
    try:
        st = os.statvfs("/dev/shm")
        if st.f_bavail * st.f_frsize > 2 * need:          # a container's /dev/shm may be tiny
            root = "/dev/shm"
    except OSError:
        pass
    path = os.path.join(root, f"fc_bench_{name}_{cfg['n']}_{cfg['m']}_{GRAPH_SEED}.fccsr")
    if world > 1:                                          # rank 0's choice of directory for everyone
        import torch.distributed as dist
        obj = [path]
        dist.broadcast_object_list(obj, src=0)
        path = obj[0]
    if rank == 0 and not os.path.exists(path):
        g = make_graph(cfg)
        tmp = path + f".{os.getpid()}.tmp"
        fc.write_similarity_binary(g, tmp)
        os.replace(tmp, path)
        del g
    barrier(world)
    hdr = np.fromfile(path, dtype="<u8", count=5)
    n, nnz = int(hdr[1]), int(hdr[2])
    if int(hdr[3]) & 1:
        raise RuntimeError("shared_graph: weighted bench graphs are not expected")
    rp = np.memmap(path, dtype="<i8", mode="r", offset=40, shape=(n + 1,))
    ci = np.memmap(path, dtype="<u4", mode="r", offset=40 + 8 * (n + 1), shape=(nnz,))
    return fc.SparseSimilarity(n, rp, ci, None, float(nnz))


def loss_hash(records, k):
    """SHA-256 of the float64 loss records of iterations 0..k (first record per iteration),
    little-endian bytes: identical bits <=> identical hash.  Both arms print it."""
    import hashlib
    seen, out = set(), []
    for it, loss in records:
        if it <= k and it not in seen:
            seen.add(it)
            out.append(loss)
    return hashlib.sha256(np.asarray(out, dtype="<f8").tobytes()).hexdigest(), len(out)


def membership_hash(x):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(x, dtype="<f8").tobytes()).hexdigest()


def bytes_model(n, nnz, c, method, weighted=False):
    """Algorithmic bytes.

    iteration: B = 8(N+1) + 12 nnz + g*8*C*nnz + s*8*C*N  with g=2, s=6 (FISTA) or g=1, s=3 (GPA)
    sweep kernel (per launch, our layout): row_ptr 8(N+1) + col 4 nnz (+8 nnz values if weighted)
       + g gathers 8*C*nnz + own row 8*C*N + xs writes g*8*C*N + prod 8 N
    """
    g = 1 if method == "gpa" else 2
    s = 3 if method == "gpa" else 6
    it = 8 * (n + 1) + 12 * nnz + g * 8 * c * nnz + s * 8 * c * n
    sweep = 8 * (n + 1) + (12 if weighted else 4) * nnz + g * 8 * c * nnz + 8 * c * n + g * 8 * c * n + 8 * n
    return it, sweep


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi takes a moment to start: wait for its first sample so a short
            # timed region still has one (taken as the region starts)
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            n0 = len(self.lines)
            t0 = time.time()
            while len(self.lines) == n0 and time.time() - t0 < 0.3:   # one sample at the region's end
                time.sleep(0.01)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                mx = float(p[2])
            except ValueError:
                continue
            for k, name in enumerate(names):
                if p[5 + k].lower() == "active":
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo", rank=rank, world_size=world)
    return world, rank, local


def allmax(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_reference_run(cfg, graph, x0, budget_s, iters_wanted, workers=0, want_x=False, sim=None):
    """The reference's own run_fista/run_gpa (oracle/_ref) on the same graph and x0, with
    `workers` threads (0 = all host cores); runs iters_wanted iterations unless a one-iteration
    probe says that exceeds budget_s.  Plain FISTA for the FISTA configs: the reference has no
    backtracking, so config B's line-search variant has no reference arm."""
    from oracle import FISTA, GPA, Reference, reference_available
    if not reference_available():
        return None
    ref = Reference()
    if workers <= 0:
        workers = ref.lib.fcref_resolve_workers(os.cpu_count() or 1)
    if sim is None:
        sim = ref.similarity(graph, fast=True)
    method = GPA if cfg["method"] == "gpa" else FISTA
    # probe: one iteration to size the sample
    t0 = time.perf_counter()
    r = sim.solve(x0, method=method, max_iter=1, fista_restart=True, workers=workers, want_x=want_x)
    probe = time.perf_counter() - t0
    el = r["elapsed_ms"]
    per_it = (el[-1] - el[0]) / 1e3 if len(el) >= 2 and el[-1] > el[0] else probe
    iters = int(max(1, min(iters_wanted, budget_s // max(per_it, 1e-9))))
    if iters > 1:
        r = sim.solve(x0, method=method, max_iter=iters, fista_restart=True, workers=workers, want_x=want_x)
        el = r["elapsed_ms"]
    t_it = (el[-1] - el[0]) / 1e3 / max(1, len(el) - 1)
    return {"s_per_iter": t_it, "iters": len(el) - 1, "cores": int(workers), "probe_s": probe,
            "records": [(it, loss) for it, loss, _ in r["records"]], "membership": r["membership"],
            "method": "gpa" if method == GPA else "fista", "sim": sim}


def run_reference_arm(args, cfg):
    """The reference's CPU solver (oracle/_ref: the unmodified reference headers) on the
    same graph, x0 and iteration count as our arm.  Loads no repo CUDA code: the graph
    comes from the host-only generator build (oracle/_build/libfcgen.so)."""
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    from oracle import Reference, reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libfcref.so not built"}))
        return 0
    t0 = time.perf_counter()
    graph = make_graph(cfg, host_only=True)
    t_graph = time.perf_counter() - t0
    ref = Reference()
    x0 = ref.init_membership(cfg["n"], cfg["c"], 0, X0_SEED, 0)
    budget = float(os.environ.get("FC_REF_BUDGET_S", "400"))
    # K iterations from x0 = the iteration count of our arm's end-to-end solve, so the two
    # parity hashes compare the same records (unless the budget cuts the run short)
    res = cpu_reference_run(cfg, graph, x0, budget, args.steps, want_x=True)
    value = 1.0 / res["s_per_iter"]
    it_b, _ = bytes_model(graph.n, graph.nnz, cfg["c"], cfg["method"])
    k = res["iters"]
    lh, nrec = loss_hash(res["records"], k)
    sample = (f"full config {args.config} graph (n={graph.n}, nnz={graph.nnz}), {k} "
              f"{res['method'].upper()} iterations of the reference run_{res['method']} from x0 = "
              f"init_membership(kRandom, seed {X0_SEED}), fista_restart=true, {res['cores']} worker threads"
              + (f" (time-bounded to ~{budget:.0f}s)" if k < args.steps else ""))
    line = {
        "impl": "reference", "metric": "fista_iterations_per_s" if cfg["method"] != "gpa" else "gpa_iterations_per_s",
        "value": value, "unit": "iter/s", "n_gpus": args.gpus, "steps": k, "warmup": 0,
        "ms_per_step": res["s_per_iter"] * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": config_name(args.config, cfg), "n": graph.n, "nnz": graph.nnz,
                   "edges_undirected": (graph.nnz - graph.n) // 2, "k": cfg["c"], "graph_gen_s": round(t_graph, 1)},
        "edges_per_s": graph.nnz * value, "achieved_gbs": it_b * value / 1e9,
        "cpu_baseline": {"value": value, "unit": "iter/s", "cores": res["cores"], "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "parity": {"method": res["method"], "iterations": k, "records": nrec, "loss_sha256": lh,
                   "membership_sha256": membership_hash(res["membership"]),
                   "final_loss": res["records"][-1][1] if res["records"] else None},
    }
    print(json.dumps(line))
    return 0


def config_name(name, cfg):
    return (f"config {name}: {cfg['kind']} n={cfg['n']}, {cfg['m']} edge draws, k={cfg['c']}, "
            f"{cfg['method'].upper()}" + (", locality on" if cfg.get("locality") else ""))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("FC_BENCH_CONFIG", "C"), choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--parity-mode", type=int, default=0, choices=[0, 1],
                    help="numerical contract of the timed solve: 0 bitwise (default), 1 tolerance mode")
    ap.add_argument("--no-tolerance-leg", action="store_true",
                    help="skip the extra tolerance-mode timing reported under 'tolerance_mode'")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference_arm(args, cfg)
    if args.warmup < 3:
        args.warmup = 3

    world, rank, local = dist_setup(args)
    import torch
    import paper_2506_04045_b200 as fc
    from paper_2506_04045_b200 import capi

    torch.cuda.set_device(local)
    t_setup = time.perf_counter()
    graph = make_graph(cfg) if world == 1 else shared_graph(cfg, args.config, rank, world)
    t_graph = time.perf_counter() - t_setup
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        obj = [capi.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    ctx = capi.Context(local, rank=rank, world=world, nccl_id=nccl_id)
    ctx.set_parity_mode(args.parity_mode)
    x0 = fc.init_membership(cfg["n"], cfg["c"], fc.InitStrategy(fc.InitKind.kRandom, X0_SEED), ctx=ctx)
    ctx.upload(graph)
    bounds = ctx.partition()
    method = {"gpa": capi.GPA, "fista": capi.FISTA, "fista_bt": capi.FISTA_BT}[cfg["method"]]
    total = args.warmup + args.steps
    step0 = 0.0
    if method == capi.FISTA_BT:
        # start from 20x the Lipschitz-safe step so the line search has work to do
        step0 = 20.0 * fc.default_step_size(graph, graph.n)
    # warm-up, the timed pass (K iterations as the library runs them: CUDA-graph replays,
    # no instrumentation), then a second pass of K iterations with per-kernel CUDA events
    # on the library's stream for the kernel breakdown and the roofline
    scfg = capi.Context.config(method=method, step_size=step0, max_iter=total + args.steps + 1, fista_restart=True)
    stream = torch.cuda.ExternalStream(ctx.stream_ptr(), device=local)

    # ---- device-resident timing --------------------------------------------------------
    ctx.begin(x0, scfg)
    ctx.run(args.warmup)
    ctx.sync()
    launches0 = ctx.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier(world)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ev0.record(stream)
        ctx.run(args.steps)
        ev1.record(stream)
        ev1.synchronize()
    torch.cuda.synchronize()
    barrier(world)
    launches = ctx.launch_count() - launches0
    ms_local = ev0.elapsed_time(ev1)
    ctx.set_profiling(True)                            # kernel-breakdown pass
    ctx.run(args.steps)
    ctx.sync()
    kt = ctx.kernel_times()
    ctx.set_profiling(False)
    done = ctx.sync()
    res = ctx.end(graph.n, cfg["c"], want_x=False)
    ms = allmax(ms_local, world)
    iters_done = res["iterations"]
    # the timed passes were real iterations iff the run got past them (a converged run makes
    # later passes no-ops); the breakdown pass is scaled by the iterations it really ran
    if not done or method == capi.FISTA_BT:            # no stop rule fired: every pass was a real iteration
        valid_count, prof_iters = True, args.steps
    else:
        valid_count = iters_done >= total
        prof_iters = max(0, min(args.steps, iters_done - total))
    value = args.steps / (ms / 1e3)

    # ---- tolerance mode (fc_set_parity_mode 1), reported beside the bitwise headline ------
    tol_leg = None
    if args.parity_mode == 0 and not args.no_tolerance_leg and cfg["c"] <= 128 and method != capi.FISTA_BT:
        ctx.set_parity_mode(1)
        ctx.begin(x0, capi.Context.config(method=method, max_iter=args.warmup + 2 * args.steps + 1,
                                          fista_restart=True))
        ctx.run(args.warmup)
        ctx.sync()
        barrier(world)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.run(args.steps)
        e1.record(stream)
        e1.synchronize()
        tms = allmax(e0.elapsed_time(e1), world)
        ctx.set_profiling(True)
        ctx.run(args.steps)
        ctx.sync()
        tkt = ctx.kernel_times()
        ctx.set_profiling(False)
        tdone = ctx.sync()
        tres = ctx.end(graph.n, cfg["c"], want_x=False)
        ctx.set_parity_mode(0)
        it_b_tol = 8 * (graph.n + 1) + 12 * graph.nnz + 8 * cfg["c"] * graph.nnz + 6 * 8 * cfg["c"] * graph.n
        tol_leg = {"value": args.steps / (tms / 1e3), "unit": "iter/s", "ms_per_step": tms / args.steps,
                   "valid": bool(not tdone or tres["iterations"] >= args.warmup + 2 * args.steps),
                   "kernel_ms_per_step": {k: v[0] / args.steps for k, v in tkt.items()},
                   "iteration_bytes": it_b_tol,
                   "achieved_gbs": it_b_tol * args.steps / (tms / 1e3) / 1e9,
                   "contract": "north star: loss 1e-9 rel per record, U 1e-7, identical supports "
                               "(single-gather FISTA by linearity + FMA contractions)"}

    # ---- end to end through the public call (host buffers) -------------------------------
    e2e = None
    if not args.no_e2e:
        ecfg = capi.Context.config(method=method, step_size=step0, max_iter=args.steps, fista_restart=True)
        # page-locked host buffers (the contract's "pinned host memory"), filled before timing;
        # the library DMAs page-locked buffers directly (pageable ones go through its staging ring)
        keep = []

        def pinned(a, view=None):
            tdt = {np.dtype(np.int64): torch.int64, np.dtype(np.float64): torch.float64,
                   np.dtype(np.uint32): torch.int32}[a.dtype]
            t = torch.empty(a.size, dtype=tdt, pin_memory=True)
            keep.append(t)
            arr = t.numpy().view(a.dtype).reshape(a.shape)
            arr[...] = a
            return arr

        g_pin = fc.SparseSimilarity(graph.n, pinned(graph.row_ptr), pinned(graph.col_idx),
                                    None if graph.values is None else pinned(graph.values), graph.frob_sq)
        x0_pin = pinned(x0)
        out_pin = pinned(np.zeros_like(x0))
        barrier(world)
        t0 = time.perf_counter()
        ctx.upload(g_pin)                              # CSR H2D (shard)
        tu = time.perf_counter()
        r = ctx.solve(x0_pin, ecfg, want_x=True, out=out_pin)   # x0 H2D, solve, membership + trace D2H
        t1 = time.perf_counter()
        e_local = t1 - t0
        e_s = allmax(e_local, world)
        lo, hi = int(bounds[rank]) if world > 1 else 0, int(bounds[rank + 1]) if world > 1 else graph.n
        csr_b = 8 * (hi - lo + 1) + 4 * int(graph.row_ptr[hi] - graph.row_ptr[lo])
        h2d = csr_b + 8 * graph.n * cfg["c"]
        d2h = 8 * graph.n * cfg["c"] + 40 * len(r["records"])
        e2e = {"value": r["iterations"] / e_s, "unit": "iter/s", "h2d_bytes_per_step": int(h2d / max(1, r["iterations"])),
               "d2h_bytes_per_step": int(d2h / max(1, r["iterations"])), "seconds": e_s,
               "iterations": r["iterations"], "upload_s": tu - t0, "solve_call_s": t1 - tu,
               "includes": "CSR upload + x0 H2D + prelude + solve + result D2H",
               "host_buffers": "page-locked (torch pin_memory), allocated and filled before the timed region"}

    # ---- parity record: `steps` plain iterations from x0 (the reference arm runs the same) ----
    parity = None
    if rank == 0 or world > 1:
        plain = capi.GPA if method == capi.GPA else capi.FISTA
        if e2e is not None and plain == method:
            pr = r
        else:
            pcfg = capi.Context.config(method=plain, max_iter=args.steps, fista_restart=True)
            pr = ctx.solve(x0, pcfg, want_x=True)
        recs = [(it, loss) for it, loss, *_ in pr["records"]]
        lh, nrec = loss_hash(recs, args.steps)
        parity = {"method": "gpa" if plain == capi.GPA else "fista", "iterations": int(pr["iterations"]),
                  "records": nrec, "loss_sha256": lh,
                  "membership_sha256": membership_hash(pr["membership"]),
                  "loss_sha256_prefix12": [loss_hash(recs, k)[0][:12] for k in range(1, args.steps + 1)],
                  "final_loss": recs[-1][1] if recs else None}

    # ---- roofline of the dominant kernel (k_sweep) -----------------------------------------
    peak, peak_kind = peaks()
    lo, hi = (int(bounds[rank]), int(bounds[rank + 1])) if world > 1 else (0, graph.n)
    nnz_l = int(graph.row_ptr[hi] - graph.row_ptr[lo])
    # tolerance mode gathers one operand per FISTA sweep (the GPA byte model)
    bm = "gpa" if args.parity_mode == 1 else cfg["method"]
    it_b_total, _ = bytes_model(graph.n, graph.nnz, cfg["c"], cfg["method"])
    if args.parity_mode == 1 and cfg["method"] != "gpa":   # one gather per sweep, six N x C streams
        it_b_total = 8 * (graph.n + 1) + 12 * graph.nnz + 8 * cfg["c"] * graph.nnz + 6 * 8 * cfg["c"] * graph.n
    _, sweep_b = bytes_model(hi - lo, nnz_l, cfg["c"], bm)
    sweep_ms, sweep_n = kt["sweep"]
    sweep_avg = sweep_ms / max(1, sweep_n)
    if prof_iters != args.steps:                       # converged during the breakdown pass: no-op launches
        sweep_avg = 0.0
    achieved = sweep_b / (sweep_avg / 1e3) / 1e9 if sweep_avg > 0 else None
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "sweep_traffic.json")) as f:
            tr = json.load(f)
        if tr.get("config") == args.config and world == 1:
            traffic = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    # FP64-issue rooflines of the step and Gram kernels (secondary: not the dominant kernel).
    # Under the bitwise contract every DADD / DMUL is one FP64 lane-op (no FMA), so the
    # ceiling is 64 FP64 lanes per SM x SMs x the SM clock.  Algorithmic ops per row:
    #   step: gradient 2C^2 + extrapolation 3C + grad/step 4C;  Gram (dual): 2 C(C+1) + 3C.
    secondary = None
    if kt is not None and prof_iters:
        try:
            props = torch.cuda.get_device_properties(local)
            sms = props.multi_processor_count
        except Exception:
            sms = 148
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                clk_max = float(json.load(f).get("sm_max_mhz", 1965.0))
        except Exception:
            clk_max = 1965.0
        fp64_peak = 64 * sms * clk_max * 1e6 / 1e12          # Tops/s of DADD / DMUL
        rows_l = hi - lo
        cc = cfg["c"]
        secondary = {}
        for name, ops_row in (("step", 2 * cc * cc + 7 * cc), ("gram", 2 * cc * (cc + 1) + 3 * cc)):
            ms_k = kt[name][0] / prof_iters if name in kt else 0.0
            if ms_k > 0:
                ach = ops_row * rows_l / (ms_k / 1e3) / 1e12
                secondary[name] = {"bound": "fp64 issue (no-FMA bitwise contract)", "achieved": ach, "peak": fp64_peak,
                                   "unit": "Tops/s", "frac": ach / fp64_peak, "ops_per_row": ops_row,
                                   "ms_per_step": ms_k,
                                   "peak_source": f"64 FP64 lanes/SM x {sms} SMs x {clk_max:.0f} MHz"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import reference_available
        if reference_available():
            budget = float(os.environ.get("FC_CPU_BUDGET_S", "30"))
            rr = cpu_reference_run(cfg, graph, x0, budget, 2, want_x=True)
            cpu = {"value": 1.0 / rr["s_per_iter"], "unit": "iter/s", "cores": rr["cores"], "kind": "reference",
                   "sample": f"{rr['iters']} {rr['method'].upper()} iteration(s) of the reference run_{rr['method']} "
                             f"on the full config {args.config} graph from the same x0 (oracle/_ref, "
                             f"{rr['cores']} threads), time-bounded to ~{budget:.0f}s"}
            # in-line parity: the same iterations on the device, compared bit for bit
            plain = capi.GPA if rr["method"] == "gpa" else capi.FISTA
            gr = ctx.solve(x0, capi.Context.config(method=plain, max_iter=rr["iters"], fista_restart=True),
                           want_x=True)
            g_recs = [(it, loss) for it, loss, *_ in gr["records"]]
            d = np.abs(gr["membership"] - rr["membership"])
            cpu["parity"] = {
                "iterations": rr["iters"],
                "loss_records_equal": loss_hash(g_recs, rr["iters"]) == loss_hash(rr["records"], rr["iters"]),
                "membership_max_abs_diff": float(d.max()) if d.size else 0.0,
                "membership_bitwise_equal": bool(np.array_equal(gr["membership"].view(np.uint64),
                                                                rr["membership"].view(np.uint64))),
                "supports_equal": bool(np.array_equal(gr["membership"] == 0, rr["membership"] == 0)),
            }
            if tol_leg is not None:                    # the tolerance mode against the same reference run
                ctx.set_parity_mode(1)
                tr = ctx.solve(x0, capi.Context.config(method=plain, max_iter=rr["iters"], fista_restart=True),
                               want_x=True)
                ctx.set_parity_mode(0)
                want = {it: loss for it, loss in rr["records"]}
                rel = max(abs(loss - want[it]) / abs(want[it]) for it, loss, *_ in tr["records"])
                tol_leg["vs_reference"] = {
                    "iterations": rr["iters"], "max_rel_loss_diff": rel,
                    "membership_max_abs_diff": float(np.abs(tr["membership"] - rr["membership"]).max()),
                    "supports_equal": bool(np.array_equal(tr["membership"] == 0, rr["membership"] == 0)),
                    "iterations_equal": int(tr["iterations"]) == rr["iters"]}
            if rr.get("sim") is not None:
                del rr["sim"]

    if rank == 0:
        step_ms = ms / args.steps
        line = {
            "metric": "fista_iterations_per_s" if cfg["method"] != "gpa" else "gpa_iterations_per_s",
            "value": value, "unit": "iter/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": config_name(args.config, cfg), "n": graph.n, "nnz": graph.nnz,
                       "edges_undirected": (graph.nnz - graph.n) // 2, "k": cfg["c"],
                       "parallelism": f"rows{world}", "l2": "inputs >> 126 MB L2 (no flush needed)",
                       "exchange": ("halo" if ctx.halo_info()[0] else "allgather") if world > 1 else None,
                       "graph_gen_s": round(t_graph, 1)},
            "edges_per_s": graph.nnz * value,
            "achieved_gbs": it_b_total * value / 1e9,
            "iteration_bytes": it_b_total,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                         "kernel": "k_sweep", "algorithmic_bytes_per_launch": sweep_b,
                         "avg_launch_ms": sweep_avg, "peak_source": peak_kind},
            "kernel_ms_per_step": ({k: v[0] / prof_iters for k, v in kt.items()} if prof_iters else None),
            "secondary_rooflines": secondary,
            "kernel_timing": "per-kernel CUDA events on the library stream, second pass of the same K iterations",
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity": parity,
            "parity_mode": args.parity_mode,
            "tolerance_mode": tol_leg,
            "clocks": clk.summary(),
            "valid": bool(valid_count),
        }
        print(json.dumps(line))
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
