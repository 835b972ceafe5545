"""GPU parity: the sm_100a product path versus the oracle and the reference's own outputs.

Every comparison is bit-exact (outputs are the unique integers in [0, p)).
Small sizes compare every entry with the exact u128 oracle or the golden
vectors produced by the reference library; large sizes use Freivalds'
check (C s == A (B s) mod p for random s), which is size-independent.
"""
import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, params=["dmma", "i8", "rns", None])
def engine(request):
    """Every test runs on every engine: the FP64 DMMA multiword engine, the
    base-256 int8 tcgen05 engine, the RNS int8 tcgen05 engine and the library
    default (None: per-shape choice between the two tcgen05 engines)."""
    F.set_default_engine(request.param)
    yield request.param
    F.set_default_engine(None)


COMBOS = [(1, 1), (1, 2), (2, 1), (1, 3), (3, 1), (1, 4), (4, 1), (2, 2), (2, 3), (3, 2), (2, 4),
          (4, 2)]


def ref_lambda(u, v, p, k):
    lam = F.mw_block_size(u, v, p)
    return None if lam is None else min(lam, max(k, 1))


def max_bits(u, v):
    """Largest bitsize whose every prime admits (u,v) (Table 3.1 rule)."""
    return F.variant_bit_limit(u, v)


def test_golden_vectors(golden):
    """Outputs of the reference library itself (tests/golden/make_golden.py)."""
    n_checked = 0
    for c in golden["cases"]:
        p, A, B = O.seeded_inputs(c["m"], c["k"], c["n"], c["bits"], c["seed"])
        Fc = F.FpContext.make(p)
        for prod in (F.mw_product, F.mw_product_workspace, F.mw_product_concat):
            C = prod(A, B, c["u"], c["v"], c["lam"], Fc)
            assert O.fnv1a64(C) == c["fnv1a64"], (prod.__name__, c)
            if "C" in c:
                assert [int(x) for x in C.ravel()] == c["C"]
            if c["m"] * c["n"] * c["k"] > 2 ** 26:
                break
        n_checked += 1
    assert n_checked == len(golden["cases"])


def test_config1_checksum(engine):
    """BASELINE config 1: 1024^3, 50-bit prime, (2,2), lambda 7 (reference C)."""
    p, A, B = O.seeded_inputs(1024, 1024, 1024, 50)
    tm = F.Timing()
    C = F.mw_product(A, B, 2, 2, 7, F.FpContext.make(p), timing=tm)
    assert C[0, 0] == 247707968029641 and C[-1, -1] == 526583644345359
    assert (C == O.exact_mod_gemm(A, B, p)).all()
    assert tm.launches == (4 if tm.engine == F.ENGINE_RNS else 3)  # packs, GEMM (+ RNS CRT)
    # exact K-block between reductions: 28 terms (DMMA, signed words), an
    # int32 segment of 147 x 64 terms (base-256, 7 digits) or 1032 x 64 (RNS)
    want = {"dmma": (28,), "i8": (9408,), "rns": (66048,), None: (9408, 66048)}[engine]
    assert tm.lambda_k in want


@pytest.mark.parametrize("u,v", COMBOS)
def test_every_word_pair_config(u, v):
    rng = np.random.default_rng(u * 10 + v)
    top = max_bits(min(u, v), max(u, v)) if (min(u, v), max(u, v)) in [(1, 1), (1, 2), (1, 3), (1, 4), (2, 2), (2, 3)] else 52
    bits_list = sorted({3, 5, min(top, 20), top - 1, top} | {int(b) for b in rng.integers(4, top + 1, 3)})
    for bits in bits_list:
        p = F.prev_prime(1 << bits)
        if p < 5 or F.mw_block_size(u, v, p) is None:
            continue
        for (m, k, n) in ((1, 1, 1), (17, 33, 9), (65, 129, 67), (130, 517, 200)):
            A = rng.integers(0, p, size=(m, k)).astype(np.float64)
            B = rng.integers(0, p, size=(k, n)).astype(np.float64)
            lam = ref_lambda(u, v, p, k)
            # exactly these words on the FP64 engine: every (u,v) kernel instantiation runs
            C = F.mw_product(A, B, u, v, lam, F.FpContext.make(p), flags=F.DMMA_EXACT_WORDS)
            assert (C == O.exact_mod_gemm(A, B, p)).all(), (u, v, bits, m, k, n)


@pytest.mark.parametrize("bits,u,v", [(26, 1, 1), (35, 1, 2), (39, 1, 3), (42, 1, 4), (48, 2, 2),
                                      (52, 2, 2), (52, 2, 3), (51, 2, 2)])
def test_worst_case_all_p_minus_1(bits, u, v):
    """All-(p-1) inputs maximise every dot product."""
    p = F.prev_prime(1 << bits)
    m, k, n = 72, 1000, 40
    for fill in (p - 1, (p - 1) // 2, (p + 1) // 2):
        A = np.full((m, k), float(fill))
        B = np.full((k, n), float(fill))
        want = (fill * fill * k) % p
        for fl in (0, F.DMMA_EXACT_WORDS):  # the engine's own word choice and exactly (u,v)
            C = F.mw_product(A, B, u, v, ref_lambda(u, v, p, k), F.FpContext.make(p), flags=fl)
            assert (C == want).all(), (bits, fill, fl)


def test_edge_shapes_and_values():
    p = F.prev_prime(1 << 45)
    Fc = F.FpContext.make(p)
    lam = ref_lambda(2, 2, p, 64)
    assert F.mw_product(np.zeros((0, 5)), np.zeros((5, 3)), 2, 2, lam, Fc).shape == (0, 3)
    assert F.mw_product(np.zeros((4, 5)), np.zeros((5, 0)), 2, 2, lam, Fc).shape == (4, 0)
    C = F.mw_product(np.zeros((4, 0)), np.zeros((0, 3)), 2, 2, lam, Fc)
    assert C.shape == (4, 3) and (C == 0).all()
    I = np.eye(50)
    B = np.random.default_rng(0).integers(0, p, size=(50, 31)).astype(np.float64)
    assert (F.mw_product(I, B, 2, 2, lam, Fc) == B).all()
    assert (F.mw_product(np.zeros((9, 50)), B, 2, 2, lam, Fc) == 0).all()


def test_strided_inputs():
    p = F.prev_prime(1 << 50)
    rng = np.random.default_rng(3)
    big = rng.integers(0, p, size=(70, 90)).astype(np.float64)
    A = big[:, 3:50]        # lda = 90
    B = big[5:52, 10:80]    # ldb = 90
    C = F.mw_product(A, B, 2, 2, 7, F.FpContext.make(p))
    assert (C == O.exact_mod_gemm(np.ascontiguousarray(A), np.ascontiguousarray(B), p)).all()


def test_tall_reduction_k262144():
    """BASELINE config 4 shape class: long K with per-block reduction (48-bit)."""
    p, A, B = O.seeded_inputs(16, 262144, 16, 48)
    C = F.mw_product(A, B, 2, 2, 31, F.FpContext.make(p))
    assert C[0, 0] == 38993103166426 and C[-1, -1] == 208543114826065
    assert (C == O.exact_mod_gemm(A, B, p)).all()


@pytest.mark.parametrize("bits", [20, 26, 30, 35, 39, 45, 52])
def test_large_freivalds(bits):
    """Full-size parity property at 4096^3 under the planner's (u,v,lambda)."""
    m = k = n = 4096
    p = F.prev_prime(1 << bits)
    A = F.random_mat(m, k, p, F.matrix_seed(1, bits, m, k, n, 0xA))
    B = F.random_mat(k, n, p, F.matrix_seed(1, bits, m, k, n, 0xB))
    pl = F.plan_for_modulus(p, m, k, n)
    C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p))
    assert O.freivalds(A, B, C, p, seed=bits, trials=2) == 0
    rows = np.arange(0, m, 511)
    cols = (rows * 7) % n
    assert [int(x) for x in O.exact_entries(A, B, p, rows, cols)] == [int(C[r, c]) for r, c in zip(rows, cols)]


def test_decompose_bit_identical_to_reference(golden):
    for d in golden["decompose"]:
        M = np.array(d["M"], dtype=np.float64).reshape(8, 16)
        wd = F.decompose(M, d["u"], F.FpContext.make(d["p"]))
        assert wd.base == d["base"]
        for i in range(d["u"]):
            assert [int(x) for x in wd.words[i].ravel()] == d["words"][i]


def test_words_products():
    p = F.prev_prime(1 << 41)
    rng = np.random.default_rng(5)
    A = rng.integers(0, p, size=(40, 77)).astype(np.float64)
    B = rng.integers(0, p, size=(77, 33)).astype(np.float64)
    Fc = F.FpContext.make(p)
    da, db = F.decompose(A, 2, Fc), F.decompose(B, 2, Fc)
    want = O.exact_mod_gemm(A, B, p)
    lam = ref_lambda(2, 2, p, 77)
    for fn in (F.mw_product_words, F.mw_product_workspace_words, F.mw_product_concat_words):
        assert (fn(da, db, 40, 77, 33, lam, Fc) == want).all()


def test_composite_modulus_workspace_and_noinverse():
    rng = np.random.default_rng(11)
    for p in (91, 100, (1 << 40) + 15, 3 * 5 * 7 * 11 * 13 * 17 * 19 * 23 * 29):
        if F.is_prime_u64(p):
            continue
        Fc = F.FpContext.make(p, allow_composite=True)
        A = rng.integers(0, p, size=(23, 45)).astype(np.float64)
        B = rng.integers(0, p, size=(45, 19)).astype(np.float64)
        u = v = 2
        lam = ref_lambda(u, v, p, 45)
        C = F.mw_product_workspace(A, B, u, v, lam, Fc)
        assert (C == O.exact_mod_gemm(A, B, p)).all()
    # plain (in-place) variant must invert alpha = word_base(100, 2) = 10: gcd 10
    Fc = F.FpContext.make(100, allow_composite=True)
    with pytest.raises(F.NoInverseError):
        F.mw_product(np.ones((2, 2)), np.ones((2, 2)), 2, 2, 1, Fc)


def test_accumulate_plugin_exact():
    """GemmKernel::accumulate contract: exact while every partial sum <= 2^53."""
    rng = np.random.default_rng(2)
    K = F.kernel_by_name("b200")
    assert K.name() == "b200"
    for (m, w, n, bound) in ((8, 4, 8, 2 ** 25), (70, 31, 45, 2 ** 20), (129, 7, 65, 2 ** 24)):
        A = rng.integers(0, bound, size=(m, w)).astype(np.float64)
        B = rng.integers(0, bound, size=(w, n)).astype(np.float64)
        C0 = rng.integers(0, 2 ** 40, size=(m, n)).astype(np.float64)
        C = C0.copy()
        K.accumulate(C, A, B)
        want = C0.astype(object) + A.astype(np.int64).astype(object).dot(B.astype(np.int64).astype(object))
        assert (C.astype(np.int64).astype(object) == want).all()


def test_block_gemm_mod():
    p = F.prev_prime(1 << 24)
    rng = np.random.default_rng(4)
    A = rng.integers(0, p, size=(33, 70)).astype(np.float64)
    B = rng.integers(0, p, size=(70, 20)).astype(np.float64)
    C = rng.integers(0, p, size=(33, 20)).astype(np.float64)
    want = (C.astype(np.int64) + O.exact_mod_gemm(A, B, p).astype(np.int64)) % p
    Fc = F.FpContext.make(p)
    F.block_gemm_mod(C, A, B, F.mw_block_size(1, 1, p), Fc)
    assert (C == want).all()


@pytest.mark.parametrize("bits", [40, 47, 52])
def test_block_gemm_mod_word_operands(bits):
    """Reference semantics above 2^26.5: word-sized operands (the way
    mw_product_words calls it, max = alpha) with the reference's lambda for
    that bound; equal to the oracle's restatement of the panel loop and to the
    exact value.  Operands >= p (below the contract bound) reduce first."""
    p = F.prev_prime(1 << bits)
    alpha = F.word_base(p, 2)
    rng = np.random.default_rng(bits)
    m, k, n = 37, 300, 29
    A = rng.integers(0, alpha + 1, size=(m, k)).astype(np.float64)
    B = rng.integers(0, alpha + 1, size=(k, n)).astype(np.float64)
    C0 = rng.integers(0, p, size=(m, n)).astype(np.float64)
    lam = F.max_block_size(alpha, alpha, p)
    assert lam is not None and lam >= 1
    Fc = F.FpContext.make(p)
    C = C0.copy()
    F.block_gemm_mod(C, A, B, lam, Fc, flags=F.CHECK_INPUTS)
    Co = C0.copy()
    assert O.lib().fo_block_gemm_mod(O._ptr(Co), O._ptr(A), k, O._ptr(B), n, m, k, n, lam, p) == 0
    want = (C0.astype(np.int64).astype(object) + A.astype(np.int64).astype(object).dot(
        B.astype(np.int64).astype(object))) % p
    assert (C == Co).all() and (C.astype(np.int64).astype(object) == want).all()
    # entries >= p: a small bound keeps the contract; every engine agrees
    A2 = A.copy()
    A2[0, :] = float(p + 5)
    B2 = rng.integers(0, 3, size=(k, n)).astype(np.float64)
    want2 = (C0.astype(np.int64).astype(object) + A2.astype(np.int64).astype(object).dot(
        B2.astype(np.int64).astype(object))) % p
    for eng in (F.ENGINE_RNS, F.ENGINE_I8, F.ENGINE_DMMA):
        C2 = C0.copy()
        F.block_gemm_mod(C2, A2, B2, 1, Fc, flags=eng)
        assert (C2.astype(np.int64).astype(object) == want2).all()
    # the contract: lambda beyond the bound (when the bound is below k), unreduced C
    if lam < k:
        with pytest.raises(F.ContractError):
            F.block_gemm_mod(C0.copy(), A, B, k, Fc, flags=F.CHECK_INPUTS)
    Cbad = C0.copy()
    Cbad[0, 0] = float(p)
    with pytest.raises(F.ContractError):
        F.block_gemm_mod(Cbad, A, B, lam, Fc, flags=F.CHECK_INPUTS)
    with pytest.raises(F.InfeasibleError):
        F.block_gemm_mod(C0.copy(), A, B, 0, Fc)


def test_check_inputs_flag():
    p = F.prev_prime(1 << 30)
    A = np.full((4, 4), float(p))  # not reduced
    with pytest.raises(F.ContractError):
        F.mw_product(A, np.ones((4, 4)), 1, 2, 1, F.FpContext.make(p), flags=F.CHECK_INPUTS)


def test_device_tensors_and_streams():
    import torch
    p = F.prev_prime(1 << 52)
    rng = np.random.default_rng(9)
    A = rng.integers(0, p, size=(300, 257)).astype(np.float64)
    B = rng.integers(0, p, size=(257, 190)).astype(np.float64)
    want = O.exact_mod_gemm(A, B, p)
    dA = torch.from_numpy(A).cuda()
    dB = torch.from_numpy(B).cuda()
    dC = torch.empty((300, 190), dtype=torch.float64, device="cuda")
    F.mw_product_device(dA, dB, dC, p, 2, 2, 1)
    assert (dC.cpu().numpy() == want).all()
    s = torch.cuda.Stream()
    dC2 = torch.zeros_like(dC)
    s.wait_stream(torch.cuda.current_stream())  # the zeroing above runs on torch's stream
    F.mw_product_device(dA, dB, dC2, p, 2, 2, 1, stream=s)
    assert (dC2.cpu().numpy() == want).all()
    # strided device views
    big = torch.from_numpy(rng.integers(0, p, size=(320, 300)).astype(np.float64)).cuda()
    sa, sb = big[:300, :257], big[:257, 20:210]
    dC3 = torch.empty((300, 190), dtype=torch.float64, device="cuda")
    F.mw_product_device(sa, sb, dC3, p, 2, 2, 1)
    assert (dC3.cpu().numpy() == O.exact_mod_gemm(sa.cpu().numpy(), sb.cpu().numpy(), p)).all()


def test_multi_gpu_in_process():
    n = F.device_count()
    if n < 2:
        pytest.skip("single GPU box")
    p, A, B = O.seeded_inputs(1000, 700, 300, 50)
    C1 = F.mw_product(A, B, 2, 2, 7, F.FpContext.make(p))
    for g in range(2, n + 1):
        assert (F.mw_product(A, B, 2, 2, 7, F.FpContext.make(p), ngpus=g) == C1).all()


def test_prepared_a_unbalanced_split_k():
    """Unbalanced scenario (m x k x 32, A's words resident and reused across
    products, driver.cpp:215-218); few output tiles force split-K."""
    import torch
    m, k, n = 1093, 3277, 32
    for bits in (20, 35, 50):
        p, A, _ = O.seeded_inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        pa = F.PreparedA(torch.from_numpy(A).cuda(), p, pl.u, pl.v)
        rng = np.random.default_rng(bits)
        for _ in range(2):
            B = rng.integers(0, p, size=(k, n)).astype(np.float64)
            dC = torch.empty((m, n), dtype=torch.float64, device="cuda")
            pa.product(torch.from_numpy(B).cuda(), dC, pl.lambda_)
            assert (dC.cpu().numpy() == O.exact_mod_gemm(A, B, p)).all(), bits
        pa.close()


def test_unbalanced_preset_full_size():
    """The paper's unbalanced preset 10923 x 32768 x 32 at 48 bits."""
    import torch
    m, k, n, bits = 10923, 32768, 32, 48
    p = F.prev_prime(1 << bits)
    dA = torch.empty((m, k), dtype=torch.float64, device="cuda")
    dB = torch.empty((k, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(dA, p, 11)
    F.random_residues_device(dB, p, 12)
    pl = F.plan_for_modulus(p, m, k, n)
    pa = F.PreparedA(dA, p, pl.u, pl.v)
    dC = torch.empty((m, n), dtype=torch.float64, device="cuda")
    pa.product(dB, dC, pl.lambda_)
    A, B, Cm = dA.cpu().numpy(), dB.cpu().numpy(), dC.cpu().numpy()
    assert O.freivalds(A, B, Cm, p, trials=2) == 0
    pa.close()


@pytest.mark.parametrize("bits,u,v,words", [(52, 2, 2, 6), (39, 1, 3, 4), (35, 1, 2, 3), (50, 2, 2, 4)])
def test_dmma_word_choice_at_lambda_collapse(engine, bits, u, v, words):
    """At the rule's lambda-collapse points the FP64 engine runs cheaper word
    counts (same C); DMMA_EXACT_WORDS keeps the caller's."""
    if engine != "dmma":
        pytest.skip("FP64 engine only")
    p = F.prev_prime(1 << bits)
    rng = np.random.default_rng(bits)
    A = rng.integers(0, p, size=(200, 300)).astype(np.float64)
    B = rng.integers(0, p, size=(300, 150)).astype(np.float64)
    want = O.exact_mod_gemm(A, B, p)
    lam = ref_lambda(u, v, p, 300)
    tm = F.Timing()
    assert (F.mw_product(A, B, u, v, lam, F.FpContext.make(p), timing=tm) == want).all()
    assert tm.engine == F.ENGINE_DMMA and tm.words == words
    tm = F.Timing()
    assert (F.mw_product(A, B, u, v, lam, F.FpContext.make(p), flags=F.DMMA_EXACT_WORDS, timing=tm) == want).all()
    assert tm.words == u * v


@pytest.mark.parametrize("bits,u,v", [(34, 1, 2), (40, 2, 2), (52, 2, 2), (52, 2, 3), (42, 1, 4)])
def test_dmma_reduction_extremes(engine, bits, u, v):
    """The in-register reduction on inputs that drive the accumulators to
    their bounds: all-(p-1), alternating (p-1)/0 columns (exact zeros next to
    maximal sums), residues near p/2 (centred words at both signs) and a zero
    A, with the engine's own word counts and exactly (u,v)."""
    if engine != "dmma":
        pytest.skip("FP64 engine only")
    p = F.prev_prime(1 << bits)
    m, k, n = 64, 2000, 72
    rng = np.random.default_rng(bits * 7 + u)
    cases = [
        (np.full((m, k), float(p - 1)), np.full((k, n), float(p - 1))),
        (np.tile([float(p - 1), 0.0], (m, k // 2)), np.tile([[float(p - 1)], [0.0]], (k // 2, n))),
        (rng.integers(p // 2 - 3, p // 2 + 4, size=(m, k)).astype(np.float64),
         rng.integers(p // 2 - 3, p // 2 + 4, size=(k, n)).astype(np.float64)),
        (np.zeros((m, k)), rng.integers(0, p, size=(k, n)).astype(np.float64)),
    ]
    for A, B in cases:
        want = O.exact_mod_gemm(A, B, p)
        for fl in (0, F.DMMA_EXACT_WORDS):
            C = F.mw_product(A, B, u, v, ref_lambda(u, v, p, k), F.FpContext.make(p), flags=fl)
            assert (C == want).all(), (bits, u, v, fl)


@pytest.mark.parametrize("bits,u,v", [(52, 2, 2), (50, 2, 2), (39, 1, 3), (26, 1, 1)])
def test_check_exactness_mode(engine, monkeypatch, bits, u, v):
    """CHECK_EXACTNESS (the reference's `check --checked` shadow replay): on
    inputs that maximise the balanced words (floor(p/2), the largest centred
    magnitude) every accumulator stays <= 2^53 at its reduction, so the
    checked product passes; with the reduction period forced past the exact
    K-block (test hook) the check fails the call with ContractError instead
    of returning a wrong C."""
    if engine != "dmma":
        pytest.skip("FP64 engine only (the int8 engines are exact by construction)")
    p = F.prev_prime(1 << bits)
    h = p // 2
    m, k, n = 64, 4096, 40
    A = np.full((m, k), float(h))
    B = np.full((k, n), float(h))
    lam = ref_lambda(u, v, p, k)
    want = (k * h * h) % p
    for fl in (0, F.DMMA_EXACT_WORDS):
        C = F.mw_product(A, B, u, v, lam, F.FpContext.make(p), flags=fl | F.CHECK_EXACTNESS)
        assert (C == want).all()
    monkeypatch.setenv("FPMM_B200_TEST_RED_EVERY", str(k // 4))  # one reduction for the whole K
    with pytest.raises(F.ContractError):
        F.mw_product(A, B, u, v, lam, F.FpContext.make(p), flags=F.DMMA_EXACT_WORDS | F.CHECK_EXACTNESS)


def test_cuda_graph_capture(engine):
    """The ASYNC device entry is stream-ordered with no host synchronisation,
    so after one warm-up call (which sizes the workspaces) a product can be
    captured in a CUDA graph and replayed: bit-identical C."""
    import torch
    m = k = n = 512
    p = F.prev_prime(1 << 50)
    pl = F.plan_for_modulus(p, m, k, n)
    A = torch.empty((m, k), dtype=torch.float64, device="cuda")
    B = torch.empty((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(A, p, 3)
    F.random_residues_device(B, p, 4)
    torch.cuda.synchronize()  # generated on torch's current stream; the product runs on s
    fl = F.ASYNC  # the fixture's default engine is added by the library binding
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
    assert O.freivalds(A.cpu().numpy(), B.cpu().numpy(), C.cpu().numpy(), p, trials=2) == 0

