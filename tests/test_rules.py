"""Host-side rule layer of the product library (C++ via the C-ABI) on CPU.

Each rule is compared with the oracle restatement and the SPEC / SURVEY
goldens; these calls never touch the GPU.
"""
import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F
from tests.test_oracle import APPENDIX_A, TABLE_3_1

VARIANTS_ALL = [(1, 1), (1, 2), (2, 1), (1, 3), (3, 1), (1, 4), (4, 1), (2, 2), (2, 3), (3, 2),
                (2, 4), (4, 2)]


def test_primes():
    for b in range(3, 63):
        assert F.prev_prime(1 << b) == O.prev_prime(1 << b)
    for n in (0, 1, 2, 3, 4, 5, 91, 97, 561, 2 ** 61 - 1, 2 ** 52 - 47, 3215031751):
        assert F.is_prime_u64(n) == O.is_prime(n), n
    assert F.prev_prime(2) == 0 and F.prev_prime(3) == 2 and F.prev_prime(9) == 7


def test_context_errors():
    F.FpContext.make(5)
    F.FpContext.make((1 << 52) - 47)
    with pytest.raises(F.Error):
        F.FpContext.make(4)
    with pytest.raises(F.Error):
        F.FpContext.make(1 << 52)
    with pytest.raises(F.Error):
        F.FpContext.make(91)
    assert not F.FpContext.make(91, allow_composite=True).prime


def test_word_base_and_bounds():
    rng = np.random.default_rng(1)
    for bits in range(3, 53):
        for p in {F.prev_prime(1 << bits), int(rng.integers(2 ** (bits - 1), 2 ** bits))}:
            for u in range(1, 5):
                assert F.word_base(p, u) == O.word_base(p, u)
                assert F.mw_block_size(1, u, p) == O.mw_block_size(1, u, p)
    assert F.word_base(97, 2) == 10 and F.word_base(101, 3) == 5
    assert F.max_block_size(2, 2, 3) == 2251799813685247
    assert F.max_block_size(0, 5, 7) == 2 ** 64 - 1


def test_table_3_1_and_rule():
    for (u, v), lim in TABLE_3_1.items():
        assert F.variant_bit_limit(u, v) == lim
    for bits, (u, v, lam) in APPENDIX_A.items():
        pl = F.plan_for_modulus(F.prev_prime(1 << bits), 8192, 8192, 8192)
        assert (pl.u, pl.v, pl.lambda_) == (u, v, lam)
    # planner equals the oracle's restatement for many shapes / thresholds
    for bits in range(2, 53):
        for (m, k, n) in ((1024, 1024, 1024), (10923, 32768, 32), (32, 100, 500), (7, 1, 7)):
            a = F.select_variant(bits, m, k, n)
            b = O.select_variant(bits, m, k, n)
            assert (a.u, a.v, a.lambda_, a.predicted_reductions, a.storage_entries) == \
                   (b.u, b.v, b.lambda_, b.reductions, b.storage)
            assert {"none": 0, "a": 1, "b": 2}[a.concat] == b.concat
    with pytest.raises(F.InfeasibleError):
        F.select_variant(53, 10, 10, 10)
    with pytest.raises(F.InfeasibleError):
        F.select_variant(40, 10, 10, 10, min_lambda=10 ** 9)


def test_kernel_block_covers_every_admitted_config():
    """The fused kernel needs an exact K-block >= 4 (one DMMA k-step) wherever
    the reference's bound admits lambda >= 1."""
    rng = np.random.default_rng(7)
    for (u, v) in VARIANTS_ALL:
        for bits in range(3, 53):
            ps = {F.prev_prime(1 << bits)}
            ps |= {F.prev_prime(int(x)) for x in rng.integers(2 ** (bits - 1) + 2, 2 ** bits, 3)}
            for p in ps:
                if p < 5 or F.bitsize(p) != bits:
                    continue
                if F.mw_block_size(u, v, p) is None:
                    continue
                lk = F.kernel_block(p, u, v)
                assert lk >= 4 and lk % 4 == 0, (u, v, p, lk)
                assert lk >= min(F.mw_block_size(u, v, p), 1 << 40) // 4 * 4 or lk >= 4


def test_random_mat_matches_reference_generator():
    for seed in (0, 1, 99):
        for p in (31, (1 << 26) - 5, (1 << 52) - 47):
            assert (F.random_mat(5, 11, p, seed) == O.random_mat(5, 11, p, seed)).all()
    assert F.matrix_seed(1, 50, 1024, 1024, 1024, 0xB) == O.matrix_seed(1, 50, 1024, 1024, 1024, 0xB)


def test_product_argument_errors_before_device():
    A = np.zeros((4, 3)); B = np.zeros((3, 5))
    with pytest.raises(F.Error):
        F.mw_product(A, np.zeros((4, 5)), 1, 1, 1, F.FpContext.make(31))
    p = (1 << 52) - 47
    with pytest.raises(F.InfeasibleError):   # lambda=2 violates lambda alpha beta + p - 1 <= 2^53
        F.mw_product(A, B, 2, 2, 2, F.FpContext.make(p))
    with pytest.raises(F.InfeasibleError):
        F.mw_product(A, B, 2, 2, 0, F.FpContext.make(p))
    with pytest.raises(F.Error):
        F.mw_product(A, B, 0, 2, 1, F.FpContext.make(p))
