"""Row-sharded exchange logic on CPU: world_size 2, gloo backend.

Each rank owns the rows `distributed.row_partition` assigns (the same rule as
tdw_problem_create), contributes its slice of the right-hand side of a step
(computed by the oracle), and the all-gather must rebuild the full vector; the
128-byte NCCL id broadcast used to bootstrap libtdw's communicator must arrive
intact.  The GPU kernels of a rank are the single-GPU kernels restricted to
its rows; this test covers the host logic around them.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, rhs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_05205_b200 import distributed as D
        ns = rhs.shape[1]
        lo, hi = D.row_partition(ns, world)[rank]
        step = 17
        full = D.gather_rows(dist, rhs[step, lo:hi], ns)
        ok_gather = np.array_equal(full, rhs[step])
        uid = bytes(range(128)) if rank == 0 else None
        got = D.broadcast_unique_id(dist, uid)
        ok_id = got == bytes(range(128))
        # max-over-ranks timing reduction used by bench.py
        t = torch.tensor([1.0 + rank])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q.put((rank, ok_gather, ok_id, float(t)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_and_bootstrap():
    from conftest import golden
    rhs = golden("march_cfg0.npz")["rhs"]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, rhs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_gather, ok_id, tmax in res:
        assert ok_gather and ok_id and tmax == 2.0, (rank, ok_gather, ok_id, tmax)
