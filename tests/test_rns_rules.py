"""Host rules of the RNS engine (rnsengine.cuh), checked on CPU.

The engine represents centred residues by their residues modulo byte moduli
and rebuilds X = sum_k a'_k b'_k mod p by the CRT in its epilogue.  These
tests pin (1) the modulus count against the exact range bound with Python
integers, (2) every CRT constant the library exports, (3) the device's
fixed-point / Shoup / Barrett reconstruction, emulated here with the same
u64 arithmetic, at the extreme values of X, and (4) the umulhi magic-number
reduction used by the packers and the epilogue.
"""
import math
import random

import numpy as np
import pytest

import paper_2601_07508_b200 as F

MASK64 = (1 << 64) - 1


def prod(xs):
    r = 1
    for x in xs:
        r *= x
    return r


@pytest.mark.parametrize("bits", [3, 8, 16, 20, 24, 25, 32, 33, 40, 41, 48, 49, 51, 52])
@pytest.mark.parametrize("k", [1, 64, 8192, 66048, 262144])
def test_modulus_count_is_minimal_and_covers_the_range(bits, k):
    p = F.prev_prime(1 << bits)
    pl = F.rns_plan(p, k)
    mods = pl["moduli"]
    h = p // 2
    assert 1000 * prod(mods) >= 2030 * k * h * h
    assert 1000 * prod(mods[:-1]) < 2030 * k * h * h or len(mods) == 1
    for i in range(len(mods)):
        for j in range(i):
            assert math.gcd(mods[i], mods[j]) == 1


def test_modulus_count_against_digit_products():
    """The point of the engine: far fewer int8 GEMMs than the D^2 digit products."""
    for bits, n_max in ((20, 7), (32, 10), (40, 12), (48, 14), (52, 15)):
        p = F.prev_prime(1 << bits)
        assert F.rns_plan(p, 8192)["n"] <= n_max
        d = (bits + 7) // 8
        assert F.rns_plan(p, 8192)["n"] < d * d or bits <= 24


@pytest.mark.parametrize("bits", [5, 20, 33, 52])
def test_crt_constants(bits):
    p = F.prev_prime(1 << bits)
    pl = F.rns_plan(p, 8192)
    mods = pl["moduli"]
    M = prod(mods)
    assert pl["Mp"] == M % p
    for i, m in enumerate(mods):
        Mi = M // m
        assert (pl["y"][i] * Mi) % m == 1
        assert pl["g"][i] == ((pl["y"][i] << 24) + m // 2) // m
        assert pl["W"][i] == (pl["y"][i] * Mi) % p


def shoup(w, p):
    return (w << 64) // p


def shoup_mulmod(t, w, ws, p):
    q = (t * ws) >> 64
    r = (t * w - q * p) & MASK64
    return r - p if r >= p else r


def barrett(x, p):
    mu = (1 << 64) // p
    q = (x * mu) >> 64
    r = (x - q * p) & MASK64
    return r - p if r >= p else r


def device_crt(X, p, pl):
    """rns_crt_kernel() on the residues of X: byte-plane dp4a sums over groups
    of four moduli, then the u64 Shoup / Barrett reconstruction."""
    planes = [0] * 10
    for m, y, W in zip(pl["moduli"], pl["y"], pl["W"]):
        r = X % m
        g = ((y << 19) + m // 2) // m
        assert g < 1 << 19 and W < 1 << 56
        for b in range(10):
            wb = (W >> (8 * b)) & 0xFF if b < 7 else (g >> (8 * (b - 7))) & 0xFF
            planes[b] += r * wb
    assert max(planes) < 1 << 32  # 32-bit dp4a accumulators
    t = (planes[8] + (planes[9] << 8) + (planes[7] >> 8) + 1024) >> 11
    f = planes[7] + (planes[8] << 8) + (planes[9] << 16)
    assert t == (f + (1 << 18)) >> 19  # the kernel's 32-bit rounding == round(F / 2^19)
    if len(pl["moduli"]) <= 16:
        S = sum(planes[b] << (8 * b) for b in range(7))
        assert S < 1 << 64
        s = barrett(S, p)
    else:
        lo = sum(planes[b] << (8 * b) for b in range(4))
        hi = sum(planes[4 + b] << (8 * b) for b in range(3))
        two32 = (1 << 32) % p
        s = barrett(shoup_mulmod(hi, two32, shoup(two32, p), p) + lo, p)
    if len(pl["moduli"]) <= 16:
        assert t * pl["Mp"] < 1 << 64
        tm = barrett(t * pl["Mp"], p)
    else:
        tm = shoup_mulmod(t, pl["Mp"], shoup(pl["Mp"], p), p)
    return s - tm if s >= tm else s + p - tm


@pytest.mark.parametrize("bits", [3, 8, 20, 25, 33, 40, 48, 52])
@pytest.mark.parametrize("k", [1, 100, 8192, 66048, 1 << 20, 1 << 26])
def test_device_crt_reconstruction_at_the_range_extremes(bits, k):
    p = F.prev_prime(1 << bits)
    pl = F.rns_plan(p, k)
    h = p // 2
    xmax = k * h * h
    rng = random.Random(bits * 1000 + k)
    cases = [0, 1, -1, xmax, -xmax, xmax - 1, -xmax + 1, h * h, -h * h]
    cases += [rng.randint(-xmax, xmax) for _ in range(300)]
    for X in cases:
        assert device_crt(X, p, pl) == X % p, X


@pytest.mark.parametrize("m", [256, 255, 253, 251, 247, 241, 217, 173])
def test_magic_reduction_exhaustive(m):
    """mod_small(s) = umulhi(s, ceil(2^32/m)) * (-m) + s (mod 2^32) for every
    s < 2^24 (the epilogue's T_hi c16 + T_lo range; the packers' dp4a sums
    stay below 2^19)."""
    magic = ((1 << 32) + m - 1) // m
    assert magic < 1 << 32 or m == 1
    s = np.arange(0, 1 << 24, dtype=np.uint64)
    q = (s * np.uint64(magic)) >> np.uint64(32)
    r = (q * np.uint64((1 << 32) - m) + s) & np.uint64(0xFFFFFFFF)
    assert np.array_equal(r, s % np.uint64(m))


def test_packer_residue_split():
    """residues16(): two dp4a over the base-256 digits of x, with the centring
    flag [x > p/2] as a ninth 'digit' weighted by the residue of -p."""
    p = F.prev_prime(1 << 52)
    pl = F.rns_plan(p, 8192)
    rng = random.Random(7)
    xs = [0, 1, p // 2, p // 2 + 1, p - 1] + [rng.randrange(p) for _ in range(2000)]
    for m in pl["moduli"]:
        w = [pow(256, j, m) for j in range(7)] + [(m - p % m) % m]
        assert all(c < 256 for c in w)
        for x in xs:
            d = [(x >> (8 * j)) & 0xFF for j in range(7)] + [1 if x > p // 2 else 0]
            s = sum(a * b for a, b in zip(d, w))
            assert s < 1 << 19
            centred = x - p if x > p // 2 else x
            assert s % m == centred % m


def test_infeasible_range_raises():
    with pytest.raises(F.InfeasibleError):
        F.rns_plan(F.prev_prime(1 << 52), 1 << 60)


@pytest.mark.parametrize("shape,bits,want", [
    ((1024, 1024, 1024), 50, "i8"),         # C1: 16 pair tiles cannot fill 74 SM pairs
    ((8192, 8192, 8192), 20, "rns"),        # C2 sweep: 7 moduli vs 9 digit products
    ((8192, 8192, 8192), 52, "rns"),        # 15 vs 49
    ((32768, 32768, 32768), 52, "rns"),     # C3
    ((4096, 262144, 4096), 48, "rns"),      # C4
    ((65536, 256, 65536), 40, "rns"),       # C5: the base-256 epilogue dominates at K = 256
    ((10923, 32768, 32), 48, "i8"),         # unbalanced: n = 32 would waste 7/8 of an RNS tile
])
def test_default_engine_choice(shape, bits, want):
    """The measured winner at each BASELINE config (profiles/round1/configs.json)."""
    m, k, n = shape
    assert F.select_engine(m, k, n, F.prev_prime(1 << bits)) == want


def test_crt_final_quotient_estimate_bound():
    """rns_crt_kernel (n <= 16): q = umulhi(S >> s, floor(2^(s+32)/p)) with
    s = max(0, bits(p) - 20) is floor(S/p) - {0, 1, 2} for every S <= 16 * 255 *
    (p - 1), so two conditional subtracts finish S mod p; and the 32-bit Shoup
    product t (M mod p) lands in [0, 2p) for t < 2^12."""
    import random
    rnd = random.Random(3)
    for bits in range(3, 53):
        p = F.prev_prime(1 << bits)
        if p < 5:
            continue
        b = (p - 1).bit_length()  # ceil(log2 p), as the host's loop computes it
        s = max(0, b - 20)
        inv = (1 << (s + 32)) // p
        assert inv < 1 << 32 and (1 << s) < p
        smax = 16 * 255 * (p - 1)
        assert smax >> s < 1 << 32
        for S in [0, 1, p - 1, p, smax, smax - 1] + [rnd.randrange(smax + 1) for _ in range(300)]:
            q = ((S >> s) * inv) >> 32
            assert 0 <= S // p - q <= 2, (bits, S)
        Mp = rnd.randrange(p)
        w = (Mp << 32) // p
        for t in [0, 1, 4095] + [rnd.randrange(4096) for _ in range(50)]:
            qt = (t * w) >> 32
            assert 0 <= t * Mp - qt * p < 2 * p


def crt_final_constants(p, pl):
    """crt_plan_final() (engine.cu): T0, C0, s2, inv2 of the one-reduction
    finalisation, or None where a bound fails (the kernel then takes the
    two-reduction path emulated by device_crt)."""
    if len(pl["moduli"]) > 16:
        return None
    gs = [((y << 19) + m // 2) // m for m, y in zip(pl["moduli"], pl["y"])]
    smax = sum((m - 1) * W for m, W in zip(pl["moduli"], pl["W"]))
    fmax = sum((m - 1) * g for m, g in zip(pl["moduli"], gs))
    t0 = (fmax + (1 << 18)) >> 19
    if t0 >= 1 << 32:
        return None
    c0 = (p - (t0 * pl["Mp"]) % p) % p
    rmax = smax + t0 * pl["Mp"] + c0
    if rmax >> 64:
        return None
    s2 = max(0, rmax.bit_length() - 31)
    if (1 << s2) >= p:
        return None
    inv2 = (1 << (s2 + 32)) // p
    if (1 << (s2 + 32)) + (rmax >> s2) * p >= p << 32:
        return None
    return {"T0": t0, "C0": c0, "s2": s2, "inv2": inv2, "rmax": rmax}


def device_crt_comb(X, p, pl, c):
    """rns_crt_spec_kernel's one-reduction finalisation on the residues of X,
    in the device's u32 / u64 arithmetic."""
    planes = [0] * 10
    for m, y, W in zip(pl["moduli"], pl["y"], pl["W"]):
        r = X % m
        g = ((y << 19) + m // 2) // m
        for b in range(10):
            wb = (W >> (8 * b)) & 0xFF if b < 7 else (g >> (8 * (b - 7))) & 0xFF
            planes[b] += r * wb
    t = (planes[8] + (planes[9] << 8) + (planes[7] >> 8) + 1024) >> 11
    assert t <= c["T0"]
    S = sum(planes[b] << (8 * b) for b in range(7))
    R = c["C0"] + S + (c["T0"] - t) * pl["Mp"]
    assert R <= c["rmax"] < 1 << 64
    q = ((R >> c["s2"]) * c["inv2"]) >> 32
    r = (R + q * ((1 << 64) - p)) & MASK64
    assert 0 <= r < 2 * p, (R, q)
    return r - p if r >= p else r


@pytest.mark.parametrize("bits", [3, 8, 20, 25, 33, 40, 48, 51, 52])
@pytest.mark.parametrize("k", [1, 256, 8192, 32768, 66048, 262144])
def test_one_reduction_crt_at_the_range_extremes(bits, k):
    """The spec CRT kernel's R = S + (T0 - t) Mp + C0 path: exact X mod p at
    the extremes of X and on random X, wherever the host enables it."""
    p = F.prev_prime(1 << bits)
    pl = F.rns_plan(p, k)
    c = crt_final_constants(p, pl)
    if c is None:
        pytest.skip("bounds fail: two-reduction path")
    h = p // 2
    xmax = k * h * h
    rng = random.Random(bits * 7 + k)
    cases = [0, 1, -1, xmax, -xmax, xmax - 1, -xmax + 1, h * h, -h * h]
    cases += [rng.randint(-xmax, xmax) for _ in range(300)]
    for X in cases:
        assert device_crt_comb(X, p, pl, c) == X % p, X


def test_one_reduction_crt_covers_the_benchmark_configs():
    """Every product the bench times takes the one-reduction path: the
    8192^3 sweep (20..52 bits) and C1, C3, C4 (per K slice), C5."""
    cfgs = [(b, 8192) for b in range(20, 53)] + [(50, 1024), (52, 32768), (48, 262144), (40, 256)]
    for bits, k in cfgs:
        p = F.prev_prime(1 << bits)
        assert crt_final_constants(p, F.rns_plan(p, k)) is not None, (bits, k)


def _fma(a, b, c):
    """fma(a, b, c) in binary64: the exact a b + c rounded once to nearest even."""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def device_crt_fp64(X, p, pl, c):
    """rns_tile_kernel's FP64 finalisation (crt4_spec<WPL, NG, true>, p <= 2^40,
    R_max < 2^53) on the residues of X, with every FP64 operation rounded as on
    the device (fma emulated exactly)."""
    planes = [0] * 10
    for m, y, W in zip(pl["moduli"], pl["y"], pl["W"]):
        r = X % m
        g = ((y << 19) + m // 2) // m
        for b in range(10):
            wb = (W >> (8 * b)) & 0xFF if b < 7 else (g >> (8 * (b - 7))) & 0xFF
            planes[b] += r * wb
    t = (planes[8] + (planes[9] << 8) + (planes[7] >> 8) + 1024) >> 11
    wpl = max(1, ((p - 1).bit_length() + 7) // 8)
    assert wpl <= 5 and all(planes[b] < 1 << 20 for b in range(wpl))
    S = float(planes[0])  # 2^52 + a - 2^52: exact for a < 2^32
    for b in range(1, wpl):
        S = _fma(float(planes[b]), float(1 << (8 * b)), S)
    ud = float(c["T0"] - t)
    R = _fma(ud, float(pl["Mp"]), S) + float(c["C0"])
    M = 6755399441055744.0
    q = _fma(R, 1.0 / float(p), M) - M
    r = _fma(-q, float(p), R)
    out = r + float(p) if r < 0.0 else r
    assert out == int(out) and 0 <= out < p
    return int(out)


@pytest.mark.parametrize("bits", [3, 8, 20, 25, 33, 38, 40])
@pytest.mark.parametrize("k", [1, 64, 256, 1024, 8192])
def test_fp64_crt_finalisation_at_the_range_extremes(bits, k):
    """The FP64-pipe finalisation rns_tile_kernel uses for p <= 2^40: exact
    X mod p at the extremes of X and on random X, wherever the host enables it
    (crt_plan_final: R_max < 2^53)."""
    p = F.prev_prime(1 << bits)
    pl = F.rns_plan(p, k)
    c = crt_final_constants(p, pl)
    if c is None or c["rmax"] >= 1 << 53 or len(pl["moduli"]) > 16:
        pytest.skip("FP64 finalisation off for this plan")
    h = p // 2
    xmax = k * h * h
    rng = random.Random(bits * 11 + k)
    cases = [0, 1, -1, xmax, -xmax, xmax - 1, -xmax + 1, h * h, -h * h]
    cases += [rng.randint(-xmax, xmax) for _ in range(150)]
    for X in cases:
        assert device_crt_fp64(X, p, pl, c) == X % p, X


def test_fp64_crt_finalisation_covers_c5():
    """C5 (k = 256, 40 bits) and the 20..40-bit short-K shapes take the FP64 path."""
    for bits in (20, 30, 40):
        p = F.prev_prime(1 << bits)
        c = crt_final_constants(p, F.rns_plan(p, 256))
        assert c is not None and c["rmax"] < 1 << 53, bits
