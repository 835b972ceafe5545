"""GPU parity of the int8 tcgen05 multiword engine (FPMM_B200_ENGINE_I8).

Same contract as the FP64 engine: C is the unique residue matrix, so every
comparison is bit-exact against the reference's outputs / the u128 oracle.
"""
import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F

pytestmark = pytest.mark.gpu
I8 = F.ENGINE_I8


def test_i8_small_exact():
    p = F.prev_prime(1 << 20)
    rng = np.random.default_rng(0)
    A = rng.integers(0, p, size=(128, 64)).astype(np.float64)
    B = rng.integers(0, p, size=(64, 32)).astype(np.float64)
    C = F.mw_product(A, B, 1, 1, 64, F.FpContext.make(p), flags=I8)
    assert (C == O.exact_mod_gemm(A, B, p)).all()


def test_i8_golden_vectors(golden):
    for c in golden["cases"]:
        p, A, B = O.seeded_inputs(c["m"], c["k"], c["n"], c["bits"], c["seed"])
        C = F.mw_product(A, B, c["u"], c["v"], c["lam"], F.FpContext.make(p), flags=I8)
        assert O.fnv1a64(C) == c["fnv1a64"], c
        if "C" in c:
            assert [int(x) for x in C.ravel()] == c["C"]


@pytest.mark.parametrize("bits", [3, 5, 8, 9, 16, 17, 20, 24, 25, 32, 33, 40, 41, 48, 49, 52])
def test_i8_every_digit_count(bits):
    p = F.prev_prime(1 << bits)
    if p < 5:
        pytest.skip("p < 5")
    pl = F.plan_for_modulus(p, 100, 100, 100)
    rng = np.random.default_rng(bits)
    for (m, k, n) in ((1, 1, 1), (17, 33, 9), (129, 65, 33), (300, 517, 70)):
        A = rng.integers(0, p, size=(m, k)).astype(np.float64)
        B = rng.integers(0, p, size=(k, n)).astype(np.float64)
        lam = min(pl.lambda_, k)
        C = F.mw_product(A, B, pl.u, pl.v, lam, F.FpContext.make(p), flags=I8)
        assert (C == O.exact_mod_gemm(A, B, p)).all(), (bits, m, k, n)


@pytest.mark.parametrize("bits", [20, 48, 52])
def test_i8_worst_case_segments(bits):
    """All-(p-1) inputs and K beyond one exact segment (forces TMEM drains)."""
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, 128, 20000, 32)
    m, k, n = 130, 20000, 40
    A = np.full((m, k), float(p - 1))
    B = np.full((k, n), float(p - 1))
    C = F.mw_product(A, B, pl.u, pl.v, min(pl.lambda_, k), F.FpContext.make(p), flags=I8)
    assert (C == ((p - 1) * (p - 1) * k) % p).all()


def test_i8_tall_reduction_k262144():
    p, A, B = O.seeded_inputs(16, 262144, 16, 48)
    C = F.mw_product(A, B, 2, 2, 31, F.FpContext.make(p), flags=I8)
    assert C[0, 0] == 38993103166426 and C[-1, -1] == 208543114826065
    assert (C == O.exact_mod_gemm(A, B, p)).all()


@pytest.mark.parametrize("bits", [20, 35, 52])
def test_i8_large_freivalds(bits):
    m = k = n = 4096
    p = F.prev_prime(1 << bits)
    A = F.random_mat(m, k, p, F.matrix_seed(1, bits, m, k, n, 0xA))
    B = F.random_mat(k, n, p, F.matrix_seed(1, bits, m, k, n, 0xB))
    pl = F.plan_for_modulus(p, m, k, n)
    C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), flags=I8)
    assert O.freivalds(A, B, C, p, seed=bits, trials=2) == 0


def test_i8_device_tensors_and_check_inputs():
    import torch
    p = F.prev_prime(1 << 45)
    rng = np.random.default_rng(3)
    A = rng.integers(0, p, size=(257, 300)).astype(np.float64)
    B = rng.integers(0, p, size=(300, 95)).astype(np.float64)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.empty((257, 95), dtype=torch.float64, device="cuda")
    F.mw_product_device(dA, dB, dC, p, 2, 2, 254, flags=I8)
    assert (dC.cpu().numpy() == O.exact_mod_gemm(A, B, p)).all()
    with pytest.raises(F.ContractError):
        F.mw_product(np.full((4, 4), float(p)), np.ones((4, 4)), 2, 2, 1, F.FpContext.make(p),
                     flags=I8 | F.CHECK_INPUTS)
