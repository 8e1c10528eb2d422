"""CPU, world_size 2 over gloo: the multi-GPU schedule of the solver, host side.

The CUDA path shards rows across ranks (fc_plan_partition: nnz-balanced, 1024-row
aligned), allgathers the new U rows after every step, and combines the per-
1024-row-block Gram / merge partials in an ORDERED chain (rank r-1 -> rank r,
then a broadcast from the last rank) so the reduction order is the reference's
ascending block order for any rank count.  This test runs exactly that schedule
with real torch.distributed (gloo) exchanges between two processes, computes the
per-shard pieces with the oracle, and checks the GPA trace and final U against
the single-process oracle bit for bit.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seq_sum(vals):
    acc = 0.0
    for v in vals:
        acc += v
    return acc


def _worker(rank, world, port, n, c, iters, q):
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import torch
        import torch.distributed as dist
        from conftest import random_graph
        from oracle import Oracle
        from paper_2506_04045_b200 import capi

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        O = Oracle()
        g = random_graph(n, 6.0, 123)
        x = O.init_random(n, c, 7)
        bounds = [int(b) for b in capi.plan_partition(g.row_ptr, world)]
        lo, hi = bounds[rank], bounds[rank + 1]
        tau = O.default_step_size(g)
        blk = 1024
        np_pairs = c * c

        def chained(partials):
            """Ordered chain: running total from rank-1, add own blocks in order, pass on, bcast."""
            run = torch.zeros(len(partials[0]) if partials else np_pairs + 1, dtype=torch.float64)
            if rank > 0:
                dist.recv(run, src=rank - 1)
            acc = run.numpy().tolist()
            for part in partials:                      # ascending block order
                acc = [a + p for a, p in zip(acc, part)]
            run = torch.tensor(acc, dtype=torch.float64)
            if rank < world - 1:
                dist.send(run, dst=rank + 1)
            dist.broadcast(run, src=world - 1)
            return run.numpy()

        loss_prev = float(n) * float(n)
        losses = []
        for it in range(iters + 1):
            xs, _ = O.fused_column_pass(x, g)           # rows are independent: each rank uses its own
            parts = []
            for b0 in range(lo, hi, blk):
                b1 = min(b0 + blk, hi)
                gb = O.share_matrix(x[b0:b1]).ravel().tolist()     # == block partial P_b
                prods = [_seq_sum([a * b for a, b in zip(xs[i].tolist(), x[i].tolist())]) for i in range(b0, b1)]
                parts.append(gb + [_seq_sum(prods)])
            tot = chained(parts)
            gmat = tot[:np_pairs].reshape(c, c)
            merge = float(tot[np_pairs])
            loss = (g.frob_sq + O.share_frob_sq(gmat)) - 2.0 * merge
            losses.append(loss)
            if loss_prev - loss <= 0.0 or it >= iters:
                break
            mine = O.gpa_step_fused(x[lo:hi], gmat, xs[lo:hi], tau)
            got = [None] * world
            dist.all_gather_object(got, mine)          # allgather of the new rows
            x = np.concatenate(got, axis=0)
            loss_prev = loss
        q.put((rank, losses, x.tobytes(), bounds))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put((rank, "ERR", traceback.format_exc(), None))


@pytest.mark.parametrize("n,c", [(5000, 4), (3000, 3)])
def test_two_rank_schedule_is_bitwise_single_process(n, c):
    import multiprocessing as mp
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from conftest import random_graph
    from oracle import GPA, Oracle

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    iters = 6
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, c, iters, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        rank, losses, xb, bounds = q.get(timeout=300)
        assert losses != "ERR", xb
        out[rank] = (losses, xb, bounds)
    for p in procs:
        p.join(timeout=60)
    assert out[0][0] == out[1][0] and out[0][1] == out[1][1]
    b = out[0][2]
    assert b[0] == 0 and b[-1] == n and b[1] % 1024 == 0 and 0 < b[1] < n

    O = Oracle()
    g = random_graph(n, 6.0, 123)
    x0 = O.init_random(n, c, 7)
    want = O.solve(g, x0, method=GPA, max_iter=iters)
    assert out[0][0] == [r[1] for r in want["records"]]
    assert np.frombuffer(out[0][1], dtype=np.float64).reshape(n, c).tobytes() == want["membership"].tobytes()


def _graph_worker(rank, world, port, q):
    try:
        sys.path.insert(0, ROOT)
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
        import hashlib
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import bench
        cfg = dict(bench.CONFIGS["A"])
        cfg["m"] = 50_000 + port % 97          # a file name no earlier run left behind
        g = bench.shared_graph(cfg, "Atest", rank, world)
        h = hashlib.sha256(np.asarray(g.row_ptr).tobytes() + np.asarray(g.col_idx).tobytes()).hexdigest()
        dist.barrier()
        q.put((rank, h, g.n, g.nnz))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e), 0, 0))


def test_bench_shared_graph_world2():
    """bench.py N > 1: rank 0 writes the graph once (FCCSR001), every rank maps the same
    bytes -- and they equal a direct generation."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_graph_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert out[0][1] == out[1][1] and len(out[0][1]) == 64, out
    sys.path.insert(0, ROOT)
    import hashlib
    import bench
    cfg = dict(bench.CONFIGS["A"])
    cfg["m"] = 50_000 + port % 97
    g = bench.make_graph(cfg)
    assert hashlib.sha256(g.row_ptr.tobytes() + g.col_idx.tobytes()).hexdigest() == out[0][1]
    import glob
    for f in glob.glob("/dev/shm/fc_bench_Atest_*") + glob.glob("/tmp/fc_bench_Atest_*"):
        os.remove(f)
