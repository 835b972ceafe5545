"""The one-process-per-GPU partitioner on a real GPU (world_size 1: only one
B200 is available to the tests).  Exercises the run-time NCCL binding,
communicator set-up, the B-word broadcast and the C gather on root."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("engine", ["i8", "rns", "dmma"])
def test_dist_world1_gather(engine):
    import torch
    import torch.distributed as td
    from paper_2601_07508_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        part = D.init_from_torch(0)
        m, k, n, bits = 300, 200, 70, 52
        p, A, B = O.seeded_inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        r0, rn = part.rows_for(m, pl.u, pl.v)
        assert (r0, rn) == (0, m)
        dA = torch.from_numpy(A).cuda()
        dB = torch.from_numpy(B).cuda()
        dCr = torch.empty((rn, n), dtype=torch.float64, device="cuda")
        dCf = torch.empty((m, n), dtype=torch.float64, device="cuda")
        eng = {"i8": F.ENGINE_I8, "rns": F.ENGINE_RNS, "dmma": F.ENGINE_DMMA}[engine]
        tm = F.Timing()
        D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf, flags=eng,
                            timing=tm)
        want = O.exact_mod_gemm(A, B, p)
        assert (dCr.cpu().numpy() == want).all()
        assert (dCf.cpu().numpy() == want).all()
        # host-buffer variant (the bench's e2e path at N > 1)
        hC = torch.empty((m, n), dtype=torch.float64).pin_memory()
        D.mw_product_host(torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory(), hC, p,
                          pl.u, pl.v, pl.lambda_, m, root=0, flags=eng)
        assert (hC.numpy() == want).all()
        D.finalize()
    finally:
        td.destroy_process_group()


def test_in_process_ngpus1_equals_default():
    p, A, B = O.seeded_inputs(257, 130, 99, 47)
    pl = F.plan_for_modulus(p, 257, 130, 99)
    C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), ngpus=1)
    assert (C == O.exact_mod_gemm(A, B, p)).all()
    with pytest.raises(F.Error):
        F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), ngpus=F.device_count() + 1)


@pytest.mark.parametrize("engine,shape,bits", [("rns", (8192, 64, 8192), 52), ("dmma", (80000, 8, 40), 20),
                                               ("i8", (8192, 64, 2048), 44), ("rns", (8192, 4100, 8192), 52)])
def test_dist_world1_chunked_gather(engine, shape, bits):
    """A rank block large enough for several row chunks: the product runs chunk
    by chunk and each chunk's C rows are shipped to root on the second stream
    (at world size 1, root's own copies).  The last case also broadcasts its
    raw B (>= 256 MB, RNS) in k-chunks packed as they land, with a ragged last
    k-chunk.  C on root equals the single-process product bitwise and passes
    Freivalds."""
    import torch
    import torch.distributed as td
    from paper_2601_07508_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        D.init_from_torch(0)
        m, k, n = shape
        p = F.prev_prime(1 << bits)
        pl = F.plan_for_modulus(p, m, k, n)
        eng = {"i8": F.ENGINE_I8, "rns": F.ENGINE_RNS, "dmma": F.ENGINE_DMMA}[engine]
        assert len(D.Partitioner.chunks_for(m, m, k, n, p, pl.u, pl.v, eng)) >= 2
        dA = torch.empty((m, k), dtype=torch.float64, device="cuda")
        dB = torch.empty((k, n), dtype=torch.float64, device="cuda")
        F.random_residues_device(dA, p, 11)
        F.random_residues_device(dB, p, 12)
        dCr = torch.empty((m, n), dtype=torch.float64, device="cuda")
        dCf = torch.full((m, n), -1.0, dtype=torch.float64, device="cuda")
        D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf, flags=eng)
        ref = torch.empty_like(dCr)
        F.mw_product_device(dA, dB, ref, p, pl.u, pl.v, pl.lambda_, flags=eng)
        torch.cuda.synchronize()
        assert torch.equal(dCr, ref) and torch.equal(dCf, ref)
        assert O.freivalds(dA.cpu().numpy(), dB.cpu().numpy(), dCf.cpu().numpy(), p, trials=2) == 0
        D.finalize()
    finally:
        td.destroy_process_group()


def test_dist_world1_pipelined_bcast_checks_inputs():
    """CHECK_INPUTS through the pipelined raw-B broadcast (RNS, B >= 256 MB):
    a non-residue in the last k-chunk of B fails the call with ContractError;
    CHECK_EXACTNESS on the same call path is accepted (RNS: nothing to check)."""
    import torch
    import torch.distributed as td
    from paper_2601_07508_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        D.init_from_torch(0)
        m, k, n, bits = 512, 4100, 8192, 52
        p = F.prev_prime(1 << bits)
        pl = F.plan_for_modulus(p, m, k, n)
        dA = torch.empty((m, k), dtype=torch.float64, device="cuda")
        dB = torch.empty((k, n), dtype=torch.float64, device="cuda")
        F.random_residues_device(dA, p, 5)
        F.random_residues_device(dB, p, 6)
        dCr = torch.empty((m, n), dtype=torch.float64, device="cuda")
        dCf = torch.empty((m, n), dtype=torch.float64, device="cuda")
        D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf,
                            flags=F.ENGINE_RNS | F.CHECK_INPUTS | F.CHECK_EXACTNESS)
        dB[k - 1, n - 1] = float(p)
        with pytest.raises(F.ContractError):
            D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf,
                                flags=F.ENGINE_RNS | F.CHECK_INPUTS)
        D.finalize()
    finally:
        td.destroy_process_group()


def test_dist_host_large_b_is_stream_ordered():
    """mw_product_host copies A and B with non_blocking H2D on torch's stream;
    the product must run after them (a 1 GiB B takes ~20 ms to land, far
    longer than the packers need to start)."""
    import torch
    import torch.distributed as td
    from paper_2601_07508_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        D.init_from_torch(0)
        m, k, n, bits = 256, 8192, 16384, 52
        p = F.prev_prime(1 << bits)
        pl = F.plan_for_modulus(p, m, k, n)
        dA = torch.empty((m, k), dtype=torch.float64, device="cuda")
        dB = torch.empty((k, n), dtype=torch.float64, device="cuda")
        F.random_residues_device(dA, p, 21)
        F.random_residues_device(dB, p, 22)
        hA, hB = dA.cpu().pin_memory(), dB.cpu().pin_memory()
        hC = torch.empty((m, n), dtype=torch.float64).pin_memory()
        for _ in range(2):
            hC.fill_(-1.0)
            D.mw_product_host(hA, hB, hC, p, pl.u, pl.v, pl.lambda_, m, root=0)
            assert F.verify_device(dA, dB, hC.cuda(), p)["ok"]
        D.finalize()
    finally:
        td.destroy_process_group()


def test_dist_gather_is_decided_by_root():
    """Every rank gathers iff root passed C_full (agreed by the call's argument
    all-reduce); argument errors fail the call before any data moves."""
    import torch
    import torch.distributed as td
    from paper_2601_07508_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_port()))
    td.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        D.init_from_torch(0)
        m, k, n, bits = 600, 300, 260, 45
        p, A, B = O.seeded_inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        want = O.exact_mod_gemm(A, B, p)
        dCr = torch.full((m, n), -1.0, dtype=torch.float64, device="cuda")
        D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0)  # no gather
        assert (dCr.cpu().numpy() == want).all()
        # a gather needs dense row blocks: strided C rows fail the call (on every rank)
        wide = torch.empty((m, n + 8), dtype=torch.float64, device="cuda")
        dCf = torch.empty((m, n), dtype=torch.float64, device="cuda")
        with pytest.raises(F.Error):
            D.mw_product_device(dA, dB, wide[:, :n], p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf)
        # ... but without a gather they are fine
        D.mw_product_device(dA, dB, wide[:, :n], p, pl.u, pl.v, pl.lambda_, m, root=0)
        assert (wide[:, :n].cpu().numpy() == want).all()
        # a bad root and an infeasible lambda are rejected, and the communicator stays usable
        with pytest.raises(F.Error):
            D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=3)
        with pytest.raises(F.InfeasibleError):
            D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, 1 << 40, m, root=0, C_full=dCf)
        D.mw_product_device(dA, dB, dCr, p, pl.u, pl.v, pl.lambda_, m, root=0, C_full=dCf)
        assert (dCf.cpu().numpy() == want).all()
        D.finalize()
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("engine,raw", [("rns", False), ("rns", True), ("i8", False), ("dmma", True)])
def test_in_process_nccl_branch_forced(monkeypatch, engine, raw):
    """FPMM_B200_INPROC_NCCL=1 runs mw_product(ngpus=1) through the
    multi-device branch (ncclCommInitAll, B broadcast as packed words or raw
    residues, per-device C rows straight to the host)."""
    monkeypatch.setenv("FPMM_B200_INPROC_NCCL", "1")
    m, k, n, bits = 700, 600, 500, 52
    p, A, B = O.seeded_inputs(m, k, n, bits)
    pl = F.plan_for_modulus(p, m, k, n)
    eng = {"i8": F.ENGINE_I8, "rns": F.ENGINE_RNS, "dmma": F.ENGINE_DMMA}[engine]
    tm = F.Timing()
    C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), ngpus=1,
                     flags=eng | (F.BCAST_RAW_B if raw else 0), timing=tm)
    assert tm.ngpus == 1 and tm.comm_ms >= 0.0
    assert (C == O.exact_mod_gemm(A, B, p)).all()
