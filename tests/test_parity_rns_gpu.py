"""GPU parity of the RNS tcgen05 engine (FPMM_B200_ENGINE_RNS).

Same contract as the other engines: C is the unique residue matrix, so every
comparison is bit-exact against the reference's outputs / the u128 oracle.
The range tests drive X = sum a'b' to +-K floor(p/2)^2, where the CRT's
rounding margin is thinnest.
"""
import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F

pytestmark = pytest.mark.gpu
RNS = F.ENGINE_RNS


def test_rns_small_exact():
    p = F.prev_prime(1 << 20)
    rng = np.random.default_rng(0)
    A = rng.integers(0, p, size=(128, 64)).astype(np.float64)
    B = rng.integers(0, p, size=(64, 256)).astype(np.float64)
    C = F.mw_product(A, B, 1, 1, 64, F.FpContext.make(p), flags=RNS)
    assert (C == O.exact_mod_gemm(A, B, p)).all()


def test_rns_golden_vectors(golden):
    for c in golden["cases"]:
        p, A, B = O.seeded_inputs(c["m"], c["k"], c["n"], c["bits"], c["seed"])
        C = F.mw_product(A, B, c["u"], c["v"], c["lam"], F.FpContext.make(p), flags=RNS)
        assert O.fnv1a64(C) == c["fnv1a64"], c
        if "C" in c:
            assert [int(x) for x in C.ravel()] == c["C"]


@pytest.mark.parametrize("bits", [3, 5, 8, 9, 16, 17, 20, 24, 25, 32, 33, 40, 41, 48, 49, 51, 52])
def test_rns_every_modulus_count(bits):
    p = F.prev_prime(1 << bits)
    if p < 5:
        pytest.skip("p < 5")
    pl = F.plan_for_modulus(p, 100, 100, 100)
    rng = np.random.default_rng(bits)
    for (m, k, n) in ((1, 1, 1), (17, 33, 9), (129, 65, 257), (300, 517, 70), (256, 1000, 512)):
        A = rng.integers(0, p, size=(m, k)).astype(np.float64)
        B = rng.integers(0, p, size=(k, n)).astype(np.float64)
        lam = min(pl.lambda_, k)
        C = F.mw_product(A, B, pl.u, pl.v, lam, F.FpContext.make(p), flags=RNS)
        assert (C == O.exact_mod_gemm(A, B, p)).all(), (bits, m, k, n)


@pytest.mark.parametrize("bits", [8, 20, 33, 48, 52])
@pytest.mark.parametrize("sign", [1, -1])
def test_rns_crt_range_extremes(bits, sign):
    """a' = b' = floor(p/2) (X = +K h^2) and a' = -b' (X = -K h^2)."""
    p = F.prev_prime(1 << bits)
    h = p // 2
    m, k, n = 130, 3000, 300
    A = np.full((m, k), float(h))
    B = np.full((k, n), float(h if sign > 0 else h + 1))  # h + 1 centres to -h
    pl = F.plan_for_modulus(p, m, k, n)
    C = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=RNS)
    want = (sign * k * h * h) % p
    assert (C == want).all()


@pytest.mark.parametrize("bits", [20, 48, 52])
def test_rns_long_k_segments(bits):
    """K beyond one exact int32 segment (66048 terms): split-major slices, CRT per slice."""
    p = F.prev_prime(1 << bits)
    m, k, n = 130, 70000, 260
    rng = np.random.default_rng(bits)
    A = rng.integers(0, p, size=(m, k)).astype(np.float64)
    B = rng.integers(0, p, size=(k, n)).astype(np.float64)
    pl = F.plan_for_modulus(p, m, k, n)
    C = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=RNS)
    assert (C == O.exact_mod_gemm(A, B, p)).all()


def test_rns_worst_case_all_max():
    p = F.prev_prime(1 << 52)
    m, k, n = 200, 20000, 300
    A = np.full((m, k), float(p - 1))
    B = np.full((k, n), float(p - 1))
    C = F.mw_product(A, B, 2, 2, 1, F.FpContext.make(p), flags=RNS)
    assert (C == ((p - 1) * (p - 1) * k) % p).all()


def test_rns_strided_device_and_split():
    """Device tensors with leading dimensions, on an explicit stream; the
    tall-skinny shape takes the split-K path."""
    import torch
    p = F.prev_prime(1 << 45)
    rng = np.random.default_rng(3)
    m, k, n = 300, 4096, 40
    A = rng.integers(0, p, size=(m, k + 5)).astype(np.float64)
    B = rng.integers(0, p, size=(k, n + 3)).astype(np.float64)
    dA = torch.from_numpy(A).cuda()[:, :k]
    dB = torch.from_numpy(B).cuda()[:, :n]
    dC = torch.zeros((m, n + 7), dtype=torch.float64, device="cuda")[:, :n]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())  # dC's zeroing runs on torch's stream
    pl = F.plan_for_modulus(p, m, k, n)
    F.mw_product_device(dA, dB, dC, p, pl.u, pl.v, pl.lambda_, stream=s, flags=RNS)
    s.synchronize()
    want = O.exact_mod_gemm(A[:, :k], B[:, :n], p)
    assert (dC.cpu().numpy() == want).all()


def test_rns_freivalds_4096():
    import torch
    p = F.prev_prime(1 << 52)
    m = k = n = 4096
    A = torch.empty((m, k), dtype=torch.float64, device="cuda")
    B = torch.empty((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(A, p, 11)
    F.random_residues_device(B, p, 12)
    F.mw_product_device(A, B, C, p, 2, 2, 1, flags=RNS)
    An, Bn, Cn = A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy()
    assert O.freivalds(An, Bn, Cn, p, trials=2) == 0
    rows = np.random.default_rng(5).integers(0, m, size=8)
    assert (Cn[rows] == O.exact_mod_gemm(An[rows], Bn, p)).all()


def test_rns_matches_other_engines():
    p = F.prev_prime(1 << 37)
    rng = np.random.default_rng(9)
    A = rng.integers(0, p, size=(333, 777)).astype(np.float64)
    B = rng.integers(0, p, size=(777, 555)).astype(np.float64)
    pl = F.plan_for_modulus(p, 333, 777, 555)
    outs = [F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), flags=e)
            for e in (F.ENGINE_RNS, F.ENGINE_I8, F.ENGINE_DMMA)]
    assert (outs[0] == outs[1]).all() and (outs[0] == outs[2]).all()


def test_concurrent_products_on_two_streams():
    """Products issued asynchronously on different streams get separate
    device workspaces (packed words, residue blocks): both results exact."""
    import torch
    rng = np.random.default_rng(21)
    runs = []
    for bits, eng in ((52, F.ENGINE_RNS), (44, F.ENGINE_RNS), (30, F.ENGINE_I8)):
        p = F.prev_prime(1 << bits)
        A = rng.integers(0, p, size=(700, 1500)).astype(np.float64)
        B = rng.integers(0, p, size=(1500, 600)).astype(np.float64)
        runs.append((p, A, B, eng))
    streams = [torch.cuda.Stream() for _ in runs]
    outs = []
    for (p, A, B, eng), s in zip(runs, streams):
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.empty((A.shape[0], B.shape[1]), dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        pl = F.plan_for_modulus(p, *A.shape, B.shape[1])
        F.mw_product_device(dA, dB, dC, p, pl.u, pl.v, pl.lambda_, stream=s, flags=eng | F.ASYNC)
        outs.append((dA, dB, dC))
    torch.cuda.synchronize()
    for (p, A, B, _), (_, _, dC) in zip(runs, outs):
        assert (dC.cpu().numpy() == O.exact_mod_gemm(A, B, p)).all()


def test_rns_row_blocks_under_a_residue_budget(monkeypatch):
    """A product whose parked residues exceed the budget runs in row blocks of
    pair tiles (here forced with a tiny budget): same C."""
    monkeypatch.setenv("FPMM_B200_RNS_RESIDUE_BUDGET", str(1 << 20))
    p = F.prev_prime(1 << 50)
    rng = np.random.default_rng(8)
    A = rng.integers(0, p, size=(1100, 700)).astype(np.float64)
    B = rng.integers(0, p, size=(700, 900)).astype(np.float64)
    tm = F.Timing()
    C = F.mw_product(A, B, 2, 2, 7, F.FpContext.make(p), flags=RNS, timing=tm)
    assert (C == O.exact_mod_gemm(A, B, p)).all()
    assert tm.launches > 4  # several GEMM + CRT pairs


@pytest.mark.parametrize("bits", [8, 20, 40, 52])
@pytest.mark.parametrize("k", [64, 256])
def test_rns_short_k_extremes(bits, k):
    """K segments of <= 258 terms (the k = 256 outer-product shape): the
    epilogue reduces each product below 2^24 without the 16-bit split.  Both
    signs of the extreme X = +-K floor(p/2)^2, plus random residues."""
    p = F.prev_prime(1 << bits)
    h = p // 2
    m, n = 300, 260
    rng = np.random.default_rng(bits + k)
    cases = [(np.full((m, k), float(h)), np.full((k, n), float(h))),
             (np.full((m, k), float(h)), np.full((k, n), float(h + 1))),
             (rng.integers(0, p, size=(m, k)).astype(np.float64), rng.integers(0, p, size=(k, n)).astype(np.float64))]
    pl = F.plan_for_modulus(p, m, k, n)
    for A, B in cases:
        C = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=RNS)
        assert (C == O.exact_mod_gemm(A, B, p)).all(), (bits, k)


@pytest.mark.parametrize("knob,value", [("FPMM_B200_RNS_FLAT", "0"), ("FPMM_B200_RNS_PACK_FP64", "0"),
                                        ("FPMM_B200_RNS_PACKB_SMEM", "1"), ("FPMM_B200_RNS_EPI_SLEEP", "256"),
                                        ("FPMM_B200_RNS_GROUP", "3"), ("FPMM_B200_RNS_TILE", "0"),
                                        ("FPMM_B200_RNS_TILE", "1"), ("FPMM_B200_RNS_TILE_STAGES", "4"),
                                        ("FPMM_B200_RNS_CRT_FP64", "0"), ("FPMM_B200_RNS_PP_PAIRS", "0"),
                                        ("FPMM_B200_RNS_PINGPONG", "0"), ("FPMM_B200_RNS_PACE", "4")])
def test_rns_tuning_knobs_same_c(monkeypatch, knob, value):
    """Every INTEGRATION.md tuning knob only changes the schedule or the
    instruction mix: C stays bit-identical to the default's (and to the oracle)."""
    rng = np.random.default_rng(11)
    for bits, (m, k, n) in ((52, (700, 900, 600)), (21, (300, 200, 520)), (40, (256, 70, 300)),
                            (40, (600, 256, 520)), (30, (300, 3000, 260))):
        p = F.prev_prime(1 << bits)
        A = rng.integers(0, p, size=(m, k)).astype(np.float64)
        B = rng.integers(0, p, size=(k, n)).astype(np.float64)
        pl = F.plan_for_modulus(p, m, k, n)
        ref = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=RNS)
        monkeypatch.setenv(knob, value)
        C = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=RNS)
        monkeypatch.delenv(knob)
        assert (C == ref).all(), (knob, bits)
        assert O.freivalds(A, B, C, p, trials=2) == 0


def test_cuda_graph_capture_tile_crt():
    """The short-K RNS path (rns_tile_kernel: residues on chip, CRT in the
    epilogue) captured in a CUDA graph and replayed: the same C as the eager
    call and as the u128 oracle."""
    import torch
    m, k, n, bits = 512, 256, 640, 40
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, m, k, n)
    A = torch.empty((m, k), dtype=torch.float64, device="cuda")
    B = torch.empty((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(A, p, 5)
    F.random_residues_device(B, p, 6)
    torch.cuda.synchronize()
    fl = F.ASYNC | F.ENGINE_RNS
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, stream=s, flags=fl)
    torch.cuda.synchronize()
    ref = C.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, stream=s, flags=fl)
    C.zero_()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(C, ref)
    want = O.exact_mod_gemm(A.cpu().numpy(), B.cpu().numpy(), p)
    assert (C.cpu().numpy() == want).all()


@pytest.mark.parametrize("bits", [20, 40])
def test_tile_crt_strided_views(bits):
    """rns_tile_kernel writes C through its leading dimension: A, B and C as
    strided views of larger device buffers (ld > cols, odd offsets), ragged
    m and n, against the u128 oracle; the bytes around C stay untouched."""
    import torch
    m, k, n = 300, 256, 200
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, m, k, n)
    Abig = torch.zeros((m, k + 40), dtype=torch.float64, device="cuda")
    Bbig = torch.zeros((k, n + 24), dtype=torch.float64, device="cuda")
    Cbig = torch.full((m + 3, n + 56), -7.0, dtype=torch.float64, device="cuda")
    A, B, Cv = Abig[:, 8:8 + k], Bbig[:, 4:4 + n], Cbig[1:1 + m, 16:16 + n]
    F.random_residues_device(Abig, p, 21)
    F.random_residues_device(Bbig, p, 22)
    F.mw_product_device(A, B, Cv, p, pl.u, pl.v, pl.lambda_, flags=RNS)
    want = O.exact_mod_gemm(A.cpu().numpy(), B.cpu().numpy(), p)
    assert (Cv.cpu().numpy() == want).all()
    untouched = Cbig.clone()
    untouched[1:1 + m, 16:16 + n] = -7.0
    assert (untouched == -7.0).all()
