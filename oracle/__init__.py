"""TEST INFRASTRUCTURE ONLY -- ctypes bindings to the CPU oracle.

``liboracle.so`` is the plain-C restatement of the reference path
(``oracle/fpmm_oracle.c``); ``_ref/libfpmm_ref.so`` is the reference library
itself compiled from ``/root/reference/proj/src`` (``oracle/Makefile``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
reference legs may import this module.  The product package
(``paper_2601_07508_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libfpmm_ref.so")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)


class Plan(C.Structure):
    _fields_ = [("u", C.c_int), ("v", C.c_int), ("lambda_", C.c_uint64), ("concat", C.c_int),
                ("products", C.c_uint64), ("reductions", C.c_uint64), ("storage", C.c_uint64)]


def build(force: bool = False) -> None:
    """Compile liboracle.so (and oracle/_ref when /root/reference exists)."""
    if force or not os.path.exists(LIB_PATH) or (
            os.path.isdir("/root/reference") and not os.path.exists(REF_PATH)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a: np.ndarray, t=_dp):
    return a.ctypes.data_as(t)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.fo_prev_prime.restype = C.c_uint64
        L.fo_prev_prime.argtypes = [C.c_uint64]
        L.fo_is_prime.argtypes = [C.c_uint64]
        L.fo_bitsize.argtypes = [C.c_uint64]
        L.fo_mix_seed.restype = C.c_uint64
        L.fo_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.fo_matrix_seed.restype = C.c_uint64
        L.fo_matrix_seed.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_uint64]
        L.fo_random_mat.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, _dp]
        L.fo_fnv1a64_f64.restype = C.c_uint64
        L.fo_fnv1a64_f64.argtypes = [_dp, C.c_int64]
        L.fo_fp_reduce.restype = C.c_double
        L.fo_fp_reduce.argtypes = [C.c_double, C.c_double, C.c_double]
        L.fo_fp_mul_reduce.restype = C.c_double
        L.fo_fp_mul_reduce.argtypes = [C.c_double, C.c_double, C.c_double, C.c_double]
        L.fo_residue_mul_mod.restype = C.c_double
        L.fo_residue_mul_mod.argtypes = [C.c_double, C.c_double, C.c_uint64]
        L.fo_mod_pow.restype = C.c_double
        L.fo_mod_pow.argtypes = [C.c_double, C.c_uint64, C.c_uint64]
        L.fo_mod_inv.argtypes = [C.c_uint64, C.c_uint64, _u64p]
        L.fo_word_base.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.fo_word_bound.restype = C.c_uint64
        L.fo_word_bound.argtypes = [C.c_uint64, C.c_int]
        L.fo_max_block_size.restype = C.c_uint64
        L.fo_max_block_size.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int]
        L.fo_mw_block_size.restype = C.c_uint64
        L.fo_mw_block_size.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int]
        L.fo_variant_bit_limit.argtypes = [C.c_int, C.c_int, C.c_int]
        L.fo_select_variant.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                        C.c_uint64, C.c_int64, C.POINTER(Plan)]
        L.fo_plan_for_modulus.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                          C.c_uint64, C.c_int64, C.POINTER(Plan)]
        L.fo_decompose.argtypes = [_dp, C.c_int64, C.c_int64, C.c_uint64, C.c_int, _dp, _u64p]
        L.fo_block_gemm_mod.argtypes = [_dp, _dp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_uint64, C.c_uint64]
        L.fo_mw_product.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int,
                                    C.c_int, C.c_uint64, C.c_int, _dp]
        L.fo_exact_mod_gemm.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, _dp,
                                        C.c_int]
        L.fo_exact_mod_gemm_colmajor.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64,
                                                 C.c_uint64, _dp]
        L.fo_exact_mod_entries.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                           _i64p, _i64p, C.c_int64, _u64p, C.c_int]
        L.fo_freivalds.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                   C.c_uint64, C.c_int, C.c_int]
        _lib = L
    return _lib


def ref():
    """The reference library (compiled from /root/reference sources), or None."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_PATH):
            try:
                build()
            except Exception:
                return None
            if not os.path.exists(REF_PATH):
                return None
        L = C.CDLL(REF_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_prev_prime.restype = C.c_uint64
        L.ref_prev_prime.argtypes = [C.c_uint64]
        L.ref_is_prime.argtypes = [C.c_uint64]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_word_base.argtypes = [C.c_uint64, C.c_int, _u64p]
        L.ref_mw_block_size.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, _u64p]
        L.ref_variant_bit_limit.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_plan_for_modulus.argtypes = [C.c_uint64, C.c_int64, C.c_int64, C.c_int64, C.c_int,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int), _u64p]
        L.ref_matrix_seed.restype = C.c_uint64
        L.ref_matrix_seed.argtypes = [C.c_uint64, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                      C.c_uint64]
        L.ref_random_mat.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, _dp]
        L.ref_decompose.argtypes = [_dp, C.c_int64, C.c_int64, C.c_uint64, C.c_int, _dp, _u64p]
        L.ref_mw_product.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64, C.c_int,
                                     C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, _dp]
        L.ref_bench_square.argtypes = [_dp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_uint64,
                                       C.c_int, C.c_int, C.c_int, C.c_int, _dp, C.POINTER(C.c_double)]
        _ref = L
    return _ref


# ----------------------------------------------------------------- helpers

def prev_prime(limit: int) -> int:
    return int(lib().fo_prev_prime(limit))


def is_prime(n: int) -> bool:
    return bool(lib().fo_is_prime(n))


def matrix_seed(seed: int, bits: int, m: int, k: int, n: int, which: int) -> int:
    return int(lib().fo_matrix_seed(seed, bits, m, k, n, which))


def random_mat(rows: int, cols: int, p: int, seed: int) -> np.ndarray:
    out = np.empty((rows, cols), dtype=np.float64)
    lib().fo_random_mat(rows, cols, p, seed, _ptr(out))
    return out


def seeded_inputs(m: int, k: int, n: int, bits: int, seed: int = 1):
    """A, B exactly as the reference driver builds them (driver.cpp:59,204-212)."""
    p = prev_prime(1 << bits)
    A = random_mat(m, k, p, matrix_seed(seed, bits, m, k, n, 0xA))
    B = random_mat(k, n, p, matrix_seed(seed, bits, m, k, n, 0xB))
    return p, A, B


def fnv1a64(C_: np.ndarray) -> str:
    C_ = np.ascontiguousarray(C_, dtype=np.float64)
    return "%016x" % lib().fo_fnv1a64_f64(_ptr(C_), C_.size)


def word_base(p: int, u: int) -> int:
    out = C.c_uint64()
    st = lib().fo_word_base(p, u, C.byref(out))
    if st:
        raise ValueError("word_base: bad arguments")
    return out.value


def mw_block_size(u: int, v: int, p: int, t: int = 53):
    l = int(lib().fo_mw_block_size(u, v, p, t))
    return None if l == 0 else l


def variant_bit_limit(u: int, v: int, t: int = 53) -> int:
    return int(lib().fo_variant_bit_limit(u, v, t))


def select_variant(bits, m, k, n, t=53, min_lambda=1, concat_threshold=256):
    pl = Plan()
    st = lib().fo_select_variant(bits, m, k, n, t, min_lambda, concat_threshold, C.byref(pl))
    if st:
        raise ValueError("select_variant status %d" % st)
    return pl


def plan_for_modulus(p, m, k, n, t=53, min_lambda=1, concat_threshold=256):
    pl = Plan()
    st = lib().fo_plan_for_modulus(p, m, k, n, t, min_lambda, concat_threshold, C.byref(pl))
    if st:
        raise ValueError("plan_for_modulus status %d" % st)
    return pl


def decompose(M: np.ndarray, p: int, u: int):
    M = np.ascontiguousarray(M, dtype=np.float64)
    words = np.empty((u,) + M.shape, dtype=np.float64)
    base = C.c_uint64()
    st = lib().fo_decompose(_ptr(M), M.shape[0], M.shape[1], p, u, _ptr(words), C.byref(base))
    if st:
        raise ValueError("decompose status %d" % st)
    return base.value, words


def mw_product(A, B, p, u, v, lam, variant=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    Cm = np.empty((m, n), dtype=np.float64)
    st = lib().fo_mw_product(_ptr(A), _ptr(B), m, k, n, p, u, v, lam, variant, _ptr(Cm))
    if st:
        raise ValueError("mw_product status %d" % st)
    return Cm


def exact_mod_gemm(A, B, p, threads=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    Cm = np.empty((m, n), dtype=np.float64)
    lib().fo_exact_mod_gemm(_ptr(A), _ptr(B), m, k, n, p, _ptr(Cm), threads)
    return Cm


def exact_mod_gemm_colmajor(A, B, p):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    Cm = np.empty((m, n), dtype=np.float64)
    lib().fo_exact_mod_gemm_colmajor(_ptr(A), _ptr(B), m, k, n, p, _ptr(Cm))
    return Cm


def exact_entries(A, B, p, rows, cols, threads=0):
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.empty(rows.size, dtype=np.uint64)
    lib().fo_exact_mod_entries(_ptr(A), _ptr(B), A.shape[0], A.shape[1], B.shape[1], p,
                               _ptr(rows, _i64p), _ptr(cols, _i64p), rows.size, _ptr(out, _u64p),
                               threads)
    return out


def freivalds(A, B, Cm, p, seed=12345, trials=2, threads=0) -> int:
    """Number of failed Freivalds trials (0 == C consistent with A B mod p)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    Cm = np.ascontiguousarray(Cm, dtype=np.float64)
    return int(lib().fo_freivalds(_ptr(A), _ptr(B), _ptr(Cm), A.shape[0], A.shape[1], B.shape[1],
                                  p, seed, trials, threads))


def ref_mw_product(A, B, p, u, v, lam, variant=0, accelerated=False, allow_composite=False):
    """Run the reference library's own mw_product (oracle/_ref)."""
    R = ref()
    if R is None:
        raise RuntimeError("reference library not built")
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = A.shape
    n = B.shape[1]
    Cm = np.empty((m, n), dtype=np.float64)
    st = R.ref_mw_product(_ptr(A), _ptr(B), m, k, n, p, u, v, lam, variant, int(accelerated),
                          int(allow_composite), _ptr(Cm))
    if st:
        raise RuntimeError("reference mw_product status %d: %s" % (st, R.ref_last_error().decode()))
    return Cm
