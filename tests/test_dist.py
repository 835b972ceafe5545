"""Multi-GPU partitioner logic on CPU (gloo, world_size 2).

The row partition is the library's own (fpmm_b200_dist_rows, C++).  The
exchange protocol of the GPU path -- rank 0 holds B and broadcasts it, each
rank multiplies its contiguous A row block, rank 0 gathers the C row blocks in
rank order -- is replayed over torch.distributed/gloo with the CPU oracle
standing in for the per-rank kernel, and must reproduce the full product.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

import oracle as O
from paper_2601_07508_b200.dist import Partitioner

COMBOS = [(1, 1), (1, 2), (2, 2), (1, 3), (2, 3)]


@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_partition_covers_rows(nranks):
    for m in (0, 1, 7, 63, 64, 65, 1000, 8192, 32768):
        for (u, v) in COMBOS:
            blocks = [Partitioner(nranks, r).rows_for(m, u, v) for r in range(nranks)]
            pos = 0
            for (r0, rn) in blocks:
                assert rn >= 0
                if rn:
                    assert r0 == pos
                    pos += rn
            assert pos == m
            # every block but the last non-empty one is a whole number of GEMM row tiles
            full = [rn for (_, rn) in blocks if rn]
            for rn in full[:-1]:
                assert rn % 256 == 0  # whole RNS pair tiles (a multiple of every engine's row tile)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m, k, n, bits = 150, 70, 40, 48
        p, A, B = O.seeded_inputs(m, k, n, bits)
        pl = O.plan_for_modulus(p, m, k, n)
        part = Partitioner(world, rank)
        r0, rn = part.rows_for(m, pl.u, pl.v)
        A_rows = torch.from_numpy(A[r0:r0 + rn].copy())
        Bt = torch.from_numpy(B.copy()) if rank == 0 else torch.zeros((k, n), dtype=torch.float64)
        td.broadcast(Bt, src=0)                                  # B (words) broadcast
        C_rows = O.mw_product(A_rows.numpy(), Bt.numpy(), p, pl.u, pl.v, pl.lambda_)
        sizes = [part.rows_for(m, pl.u, pl.v, r)[1] for r in range(world)]
        maxr = max(sizes)
        pad = torch.zeros((maxr, n), dtype=torch.float64)
        pad[:rn] = torch.from_numpy(C_rows)
        bufs = [torch.zeros_like(pad) for _ in range(world)] if rank == 0 else None
        td.gather(pad, bufs, dst=0)                              # C row blocks -> root
        if rank == 0:
            Cfull = np.concatenate([bufs[r][:sizes[r]].numpy() for r in range(world)])
            q.put(bool((Cfull == O.exact_mod_gemm(A, B, p)).all()))
    finally:
        td.destroy_process_group()


def test_two_rank_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    assert q.get(timeout=5) is True
