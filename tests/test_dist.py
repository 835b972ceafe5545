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


def test_gather_chunks_geometry():
    """fpmm_b200_dist_chunks: consecutive whole row tiles covering the block,
    at most FPMM_B200_DIST_MAX_CHUNKS, one chunk when the block is small."""
    import paper_2601_07508_b200 as F
    for bits, (m, k, n), flags in ((20, (160000, 4, 40), F.ENGINE_DMMA), (52, (32768, 32768, 32768), 0),
                                   (52, (32768, 32768, 32768), F.ENGINE_I8), (40, (8192, 8192, 8192), 0)):
        p = F.prev_prime(1 << bits)
        for rows in (0, 1, 255, 4096, m // 8, m // 2, m):
            ch = Partitioner.chunks_for(rows, m, k, n, p, 2, 2, flags)
            assert len(ch) <= 4 and (rows == 0) == (len(ch) == 0)
            pos = 0
            for (s, ln) in ch:
                assert s == pos and ln > 0
                pos += ln
            assert pos == rows
            for (s, ln) in ch[:-1]:
                assert ln % 32 == 0
    # 8 ranks of the 32768^3 config: 4096 rows per rank run as 4 overlapped chunks
    p = F.prev_prime(1 << 52)
    assert len(Partitioner.chunks_for(4096, 32768, 32768, 32768, p, 2, 2, 0)) == 4


def _chunk_worker(rank, world, port, q):
    """The gathered product's exchange with row chunks: chunk c of every rank
    reaches root in round c (root posts one receive per rank per round, ranks
    with fewer chunks skip rounds), as dist_product_device issues them."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2601_07508_b200 as F
        m, k, n, bits = 170000, 4, 40, 20
        p = O.prev_prime(1 << bits)
        rng = np.random.default_rng(5)
        A = rng.integers(0, p, size=(m, k)).astype(np.float64)
        B = rng.integers(0, p, size=(k, n)).astype(np.float64)
        flags = F.ENGINE_DMMA
        part = Partitioner(world, rank)
        blocks = [part.rows_for(m, 1, 1, r) for r in range(world)]
        chunks = [Partitioner.chunks_for(blocks[r][1], m, k, n, p, 1, 1, flags) for r in range(world)]
        r0, rn = blocks[rank]
        C_rows = (A[r0:r0 + rn].astype(object).dot(B.astype(object)) % p).astype(np.float64)
        rounds = max(len(c) for c in chunks)
        if rank == 0:
            Cfull = np.zeros((m, n))
            Cfull[r0:r0 + rn] = C_rows
            for ci in range(rounds):
                for r in range(1, world):
                    if ci < len(chunks[r]):
                        s, ln = chunks[r][ci]
                        buf = torch.zeros((ln, n), dtype=torch.float64)
                        td.recv(buf, src=r)
                        Cfull[blocks[r][0] + s:blocks[r][0] + s + ln] = buf.numpy()
            want = (A.astype(object).dot(B.astype(object)) % p).astype(np.float64)
            q.put((bool((Cfull == want).all()), [len(c) for c in chunks]))
        else:
            for ci in range(len(chunks[rank])):
                s, ln = chunks[rank][ci]
                td.send(torch.from_numpy(np.ascontiguousarray(C_rows[s:s + ln])), dst=0)
    finally:
        td.destroy_process_group()


def test_chunked_gather_protocol_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_chunk_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
        assert pr.exitcode == 0
    ok, counts = q.get(timeout=5)
    assert ok and counts[0] >= 2  # the multi-chunk path is the one exercised
