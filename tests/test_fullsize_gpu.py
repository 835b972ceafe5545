"""Parity at the sizes BASELINE.json names.

The CPU oracle cannot recompute a 32768^3 product, so full-size outputs are
checked exactly on the device (fpmm_b200_verify_device: C in [0, p), two
Freivalds trials mod p, sampled exact entries -- the analogue of the
reference's oracle-equivalence suite, driver.cpp:37-140), and a few entries
are recomputed independently on the CPU with the u128 oracle
(oracle.exact_entries) from rows of A and columns of B copied to the host.
These shapes reach paths the small tests never do: RNS row blocks above the
residue budget (C3), split-K slices at k = 262144 (C4), the k = 256 outer
product with 65536^2 outputs (C5), and the 8192^3 modulus counts of every
sweep bitsize (C2).
"""
import numpy as np
import pytest

import oracle as O
import paper_2601_07508_b200 as F

pytestmark = pytest.mark.gpu


def _inputs(m, k, n, bits, seed=1):
    import torch
    p = F.prev_prime(1 << bits)
    A = torch.empty((m, k), dtype=torch.float64, device="cuda")
    B = torch.empty((k, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(A, p, F.matrix_seed(seed, bits, m, k, n, 0xA))
    F.random_residues_device(B, p, F.matrix_seed(seed, bits, m, k, n, 0xB))
    return p, A, B


def _cpu_entries(A, B, Cm, p, count=6, seed=3):
    """Entries recomputed on the host by the u128 oracle from A's rows and B's columns."""
    import torch
    m, k = A.shape
    n = B.shape[1]
    rng = np.random.default_rng(seed)
    rows = np.concatenate([[0, m - 1], rng.integers(0, m, size=count)]).astype(np.int64)
    cols = np.concatenate([[n - 1, 0], rng.integers(0, n, size=count)]).astype(np.int64)
    Ar = A[torch.from_numpy(rows).cuda()].cpu().numpy()
    Bc = B[:, torch.from_numpy(cols).cuda()].cpu().numpy()
    want = O.exact_entries(Ar, Bc, p, np.arange(len(rows)), np.arange(len(cols)))
    got = Cm[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()].cpu().numpy()
    return np.array_equal(np.asarray(want, dtype=np.float64), got)


def _check(A, B, Cm, p, seed=7):
    r = F.verify_device(A, B, Cm, p, seed=seed, trials=2, samples=64)
    assert r["ok"], r
    assert _cpu_entries(A, B, Cm, p)


def test_verifier_catches_corruption():
    """The device verifier flags a single wrong entry, an entry off by p and a
    non-integer, and passes the correct product."""
    import torch
    p, A, B = _inputs(640, 520, 700, 50)
    Cm = torch.empty((640, 700), dtype=torch.float64, device="cuda")
    pl = F.plan_for_modulus(p, 640, 520, 700)
    F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_)
    assert F.verify_device(A, B, Cm, p)["ok"]
    assert _cpu_entries(A, B, Cm, p)
    for (i, j, delta) in ((333, 444, 1.0), (0, 699, float(p)), (639, 0, 0.5)):
        bad = Cm.clone()
        bad[i, j] = (bad[i, j] + delta) if delta != float(p) else bad[i, j] + p
        r = F.verify_device(A, B, bad, p, trials=2, samples=8)
        assert not r["ok"], (i, j, r)
        if delta == 1.0:
            assert r["freivalds_rows"] == 2 and r["range"] == 0  # one row differs, in both trials
        else:
            assert r["range"] == 1
    # a corrupted corner is also caught by the sampled exact entries (corners first)
    bad = Cm.clone()
    bad[639, 699] = (bad[639, 699] + 3) % p
    r = F.verify_device(A, B, bad, p, trials=0, samples=4)
    assert r["samples_bad"] == 1 and r["first_bad"] == (639, 699)


def test_sweep_8192_every_bitsize():
    """C2: m = n = k = 8192, every bitsize 20..52 with the rule's (u,v,lambda),
    on the library default engine -- the products bench.py times."""
    import torch
    m = k = n = 8192
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for bits in range(20, 53):
        p, A, B = _inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_)
        r = F.verify_device(A, B, Cm, p, seed=bits, trials=2, samples=32)
        assert r["ok"], (bits, r)
        del A, B
    assert _cpu_entries(*_inputs(m, k, n, 52)[1:], Cm, F.prev_prime(1 << 52))


@pytest.mark.parametrize("engine", ["i8", "dmma"])
def test_sweep_8192_other_engines_sampled(engine):
    """The other two engines at 8192^3 on the sweep's extreme and middle bitsizes."""
    import torch
    m = k = n = 8192
    eng = {"i8": F.ENGINE_I8, "dmma": F.ENGINE_DMMA}[engine]
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for bits in (20, 35, 52):
        p, A, B = _inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_, flags=eng)
        assert F.verify_device(A, B, Cm, p, seed=bits)["ok"], bits


def test_c3_32768_cubed_52bit():
    """C3: 32768^3, 52-bit prime, rule (2,2), lambda = 1, default engine.  The
    RNS residue scratch exceeds the budget here, so the product runs in row
    blocks; 32768 terms need the plan's larger modulus count."""
    import torch
    m = k = n = 32768
    p, A, B = _inputs(m, k, n, 52)
    pl = F.plan_for_modulus(p, m, k, n)
    assert (pl.u, pl.v, pl.lambda_) == (2, 2, 1)
    assert F.rns_plan(p, k)["n"] > F.rns_plan(p, 8192)["n"]
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    tm = F.Timing()
    F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_, timing=tm)
    _check(A, B, Cm, p)


def test_c3_row_blocks_forced(monkeypatch):
    """C3's shape class with the residue budget forced small (many row blocks
    of the parked-residue path, ragged last block) equals one launch bitwise."""
    import torch
    m, k, n = 8192 + 300, 32768, 4096
    p, A, B = _inputs(m, k, n, 52)
    pl = F.plan_for_modulus(p, m, k, n)
    C1 = torch.empty((m, n), dtype=torch.float64, device="cuda")
    C2 = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.mw_product_device(A, B, C1, p, pl.u, pl.v, pl.lambda_, flags=F.ENGINE_RNS)
    monkeypatch.setenv("FPMM_B200_RNS_RESIDUE_BUDGET", str(300 << 20))
    F.mw_product_device(A, B, C2, p, pl.u, pl.v, pl.lambda_, flags=F.ENGINE_RNS)
    assert torch.equal(C1, C2)
    _check(A, B, C2, p)


@pytest.mark.parametrize("shape,bits", [((8192, 8192, 8192), 20), ((8192, 8192, 8192), 52), ((1000, 3000, 777), 45),
                                        ((65536, 256, 4096), 40), ((300, 100000, 5000), 33), ((5000, 64, 300), 26),
                                        ((4096, 256, 4096), 52), ((2000, 60000, 1000), 50), ((513, 129, 385), 8)])
def test_rns_tile_crt_equals_parked(monkeypatch, shape, bits):
    """rns_tile_kernel (residues kept on chip, CRT in the epilogue, 256 x 128
    tiles) gives the parked-residue path's C bitwise, forced on wherever it
    applies (FPMM_B200_RNS_TILE=1): full and ragged tiles, n = 4..16 moduli
    (shared-memory and TMEM residue planes), k up to one exact segment, and a
    split-K shape that keeps the parked path."""
    import torch
    m, k, n = shape
    p, A, B = _inputs(m, k, n, bits)
    pl = F.plan_for_modulus(p, m, k, n)
    C1 = torch.full((m, n), -1.0, dtype=torch.float64, device="cuda")
    C2 = torch.full((m, n), -2.0, dtype=torch.float64, device="cuda")
    monkeypatch.setenv("FPMM_B200_RNS_TILE", "1")
    F.mw_product_device(A, B, C1, p, pl.u, pl.v, pl.lambda_, flags=F.ENGINE_RNS)
    monkeypatch.setenv("FPMM_B200_RNS_TILE", "0")
    F.mw_product_device(A, B, C2, p, pl.u, pl.v, pl.lambda_, flags=F.ENGINE_RNS)
    assert torch.equal(C1, C2)
    assert F.verify_device(A, B, C1, p)["ok"]


def test_c4_tall_reduction_48bit():
    """C4: 4096 x 262144 x 4096, 48-bit prime, rule (2,2), lambda = 31: K is
    split into exact int32 slices whose residues are combined."""
    import torch
    m, k, n = 4096, 262144, 4096
    p, A, B = _inputs(m, k, n, 48)
    pl = F.plan_for_modulus(p, m, k, n)
    assert (pl.u, pl.v, pl.lambda_) == (2, 2, 31)
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    for eng in (0, F.ENGINE_I8):
        Cm.fill_(-1.0)
        F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_, flags=eng)
        _check(A, B, Cm, p)


def test_c5_outer_product_40bit():
    """C5: 65536 x 256 x 65536, 40-bit prime, rule (2,2), lambda = 256."""
    import torch
    m, k, n = 65536, 256, 65536
    p, A, B = _inputs(m, k, n, 40)
    pl = F.plan_for_modulus(p, m, k, n)
    assert (pl.u, pl.v, pl.lambda_) == (2, 2, 256)
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.mw_product_device(A, B, Cm, p, pl.u, pl.v, pl.lambda_)
    _check(A, B, Cm, p)


def test_c1_device_entry_every_engine():
    """C1 (1024^3, 50-bit, (2,2), lambda = 7) through the device entry on the
    reference's own seeded inputs, every engine: the full u128 oracle product
    and the device verifier agree."""
    import torch
    m = k = n = 1024
    bits = 50
    p, A, B = O.seeded_inputs(m, k, n, bits)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    Cm = torch.empty((m, n), dtype=torch.float64, device="cuda")
    pl = F.plan_for_modulus(p, m, k, n)
    for eng in (0, F.ENGINE_RNS, F.ENGINE_I8, F.ENGINE_DMMA):
        F.mw_product_device(dA, dB, Cm, p, pl.u, pl.v, pl.lambda_, flags=eng)
        assert F.verify_device(dA, dB, Cm, p)["ok"]
        got = Cm.cpu().numpy()
        assert (got == O.exact_mod_gemm(A, B, p)).all()
