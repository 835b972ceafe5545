"""B200-native multiword modular matrix product (arXiv 2601.07508).

Python mirror of the reference library's interface for the hot path
(``/root/reference/proj/include/fpmm``): the same names, argument order and
error behaviour, over the C-ABI in ``include/fpmm_b200.h`` implemented by the
in-tree ``libfpmm_b200.so`` (hand-written sm_100a CUDA + NCCL).

Matrices are numpy ``float64`` 2-D arrays (row-major, exactly the reference's
``Mat<double>`` layout) holding integers; device entry points take torch CUDA
tensors.  There is no CPU fallback: if the shared library is missing every
call raises, and on a machine without a GPU the device entry points raise
``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

__all__ = [
    "Error", "InfeasibleError", "NoInverseError", "ContractError", "CudaError", "NcclError",
    "FpContext", "WordDecomposition", "ProductPlan", "Variant", "kVariants", "Timing",
    "is_prime_u64", "prev_prime", "bitsize", "word_base", "word_bound", "max_block_size",
    "mw_block_size", "variant_bit_limit", "variant_admits_bits", "select_variant",
    "plan_for_modulus", "finish_plan", "kernel_block", "rns_plan", "select_engine", "mix_seed", "matrix_seed", "random_mat",
    "decompose", "mw_product", "mw_product_words", "mw_product_workspace",
    "mw_product_workspace_words", "mw_product_concat", "mw_product_concat_words",
    "block_gemm_mod", "GemmKernel", "kernel_by_name", "b200_kernel", "mw_product_device",
    "decompose_device", "accumulate_device", "verify_device", "device_count", "finalize", "lib", "LIB_PATH",
]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FPMM_B200_LIB") or os.path.join(HERE, "libfpmm_b200.so")
T = 53  # FpContext<double>::t


# ------------------------------------------------------------------ errors
class Error(RuntimeError):
    """fpmm::Error (errors.hpp:9-12)."""


class ContractError(Error):
    """fpmm::ContractError (errors.hpp:17-19)."""


class InfeasibleError(Error):
    """fpmm::InfeasibleError (errors.hpp:22-25)."""


class NoInverseError(Error):
    """fpmm::NoInverseError (errors.hpp:29-31)."""


class CudaError(Error):
    """CUDA failure on the device path (no CPU fallback exists)."""


class NcclError(Error):
    """NCCL failure in the partitioner."""


_ERRS = {1: Error, 2: InfeasibleError, 3: NoInverseError, 4: ContractError, 10: CudaError,
         11: NcclError, 12: CudaError}

ALLOW_COMPOSITE = 0x1
CHECK_INPUTS = 0x2
INPLACE_INVERSES = 0x4
BCAST_RAW_B = 0x8
ENGINE_DMMA = 0x10  # FP64 multiword on the FP64 tensor pipe (DMMA)
ENGINE_I8 = 0x20    # base-256 multiword on tcgen05.mma.kind::i8 (TMEM int32 accumulators)
ENGINE_RNS = 0x40   # byte residues mod coprime m_i <= 256, one kind::i8 GEMM per modulus, then the CRT (on chip at short K)
DMMA_EXACT_WORDS = 0x80  # FP64 engine: exactly the caller's (u,v) words (default may pick cheaper counts)
ASYNC = 0x100
CHECK_EXACTNESS = 0x200  # FP64 engine: verify every accumulator <= 2^53 at each reduction (shadow-replay analogue)
PLAIN, WORKSPACE, CONCAT = 0, 1, 2
_ENGINE_MASK = ENGINE_DMMA | ENGINE_I8 | ENGINE_RNS
_default_engine_flags = 0


def set_default_engine(name: Optional[str]) -> None:
    """Engine used when a call passes no ENGINE_* flag: "i8", "rns", "dmma" or
    None (the library default: i8 or rns by a per-shape time model)."""
    global _default_engine_flags
    _default_engine_flags = {"i8": ENGINE_I8, "rns": ENGINE_RNS, "dmma": ENGINE_DMMA, None: 0}[name]


def _eng(flags: int) -> int:
    return flags if flags & _ENGINE_MASK else flags | _default_engine_flags


class _Plan(C.Structure):
    _fields_ = [("u", C.c_int), ("v", C.c_int), ("lambda_", C.c_uint64), ("concat", C.c_int),
                ("predicted_products", C.c_uint64), ("predicted_reductions", C.c_uint64),
                ("storage_entries", C.c_uint64)]


class Timing(C.Structure):
    """fpmm_b200_timing: CUDA-event phase times of one call (ms)."""
    _fields_ = [("h2d_ms", C.c_double), ("pack_ms", C.c_double), ("gemm_ms", C.c_double),
                ("comm_ms", C.c_double), ("d2h_ms", C.c_double), ("total_ms", C.c_double),
                ("lambda_k", C.c_int64), ("launches", C.c_int32), ("ngpus", C.c_int32),
                ("engine", C.c_int32), ("words", C.c_int32), ("recon_ms", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_lib = None


def lib():
    """Load libfpmm_b200.so (built by ``__graft_entry__.build()``); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            "libfpmm_b200.so not built (%s); run python -c 'import __graft_entry__ as g; g.build()'"
            % LIB_PATH)
    L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    i32, i64, u64, vp = C.c_int, C.c_int64, C.c_uint64, C.c_void_p
    sig = {
        "fpmm_b200_last_error": (C.c_char_p, []),
        "fpmm_b200_version": (i32, []),
        "fpmm_b200_device_count": (i32, [C.POINTER(i32)]),
        "fpmm_b200_is_prime": (i32, [u64]),
        "fpmm_b200_prev_prime": (u64, [u64]),
        "fpmm_b200_context_check": (i32, [u64, i32]),
        "fpmm_b200_word_base": (i32, [u64, i32, _u64p]),
        "fpmm_b200_max_block_size": (i32, [u64, u64, u64, i32, _u64p]),
        "fpmm_b200_mw_block_size": (i32, [i32, i32, u64, i32, _u64p]),
        "fpmm_b200_variant_bit_limit": (i32, [i32, i32, i32, C.POINTER(i32)]),
        "fpmm_b200_select_variant": (i32, [i32, i64, i64, i64, i32, u64, i64, C.POINTER(_Plan)]),
        "fpmm_b200_plan_for_modulus": (i32, [u64, i64, i64, i64, i32, u64, i64, C.POINTER(_Plan)]),
        "fpmm_b200_finish_plan": (i32, [C.POINTER(_Plan), i64, i64, i64]),
        "fpmm_b200_kernel_block": (i32, [u64, i32, i32, _i64p]),
        "fpmm_b200_rns_plan": (i32, [u64, i64, C.POINTER(i32), vp, vp, vp, vp, _u64p]),
        "fpmm_b200_select_engine": (i32, [i64, i64, i64, u64, C.POINTER(C.c_uint)]),
        "fpmm_b200_mix_seed": (u64, [u64, u64]),
        "fpmm_b200_matrix_seed": (u64, [u64, i32, i64, i64, i64, u64]),
        "fpmm_b200_random_mat": (i32, [i64, i64, u64, u64, _dp]),
        "fpmm_b200_mw_product": (i32, [_dp, i64, _dp, i64, _dp, i64, i64, i64, i64, u64, i32, i32,
                                       u64, i32, i32, C.c_uint, C.POINTER(Timing)]),
        "fpmm_b200_mw_product_words": (i32, [_dp, i64, i64, u64, i32, _dp, i64, i64, u64, i32, _dp,
                                             i64, i64, i64, i64, u64, u64, i32, C.c_uint,
                                             C.POINTER(Timing)]),
        "fpmm_b200_decompose": (i32, [_dp, i64, i64, i64, u64, i32, _dp, i64, _u64p]),
        "fpmm_b200_block_gemm_mod": (i32, [_dp, i64, _dp, i64, _dp, i64, i64, i64, i64, u64, u64,
                                           C.c_uint]),
        "fpmm_b200_accumulate": (i32, [_dp, i64, _dp, i64, _dp, i64, i64, i64, i64]),
        "fpmm_b200_mw_product_device": (i32, [vp, i64, vp, i64, vp, i64, i64, i64, i64, u64, i32,
                                              i32, u64, i32, i32, vp, C.c_uint, C.POINTER(Timing)]),
        "fpmm_b200_decompose_device": (i32, [vp, i64, i64, i64, u64, i32, vp, i64, _u64p, i32, vp]),
        "fpmm_b200_accumulate_device": (i32, [vp, i64, vp, i64, vp, i64, i64, i64, i64, i32, vp]),
        "fpmm_b200_nccl_id_size": (i32, []),
        "fpmm_b200_nccl_get_unique_id": (i32, [vp]),
        "fpmm_b200_dist_init": (i32, [vp, i32, i32, i32]),
        "fpmm_b200_dist_finalize": (i32, []),
        "fpmm_b200_dist_rows": (i32, [i64, i32, i32, i32, i32, _i64p, _i64p]),
        "fpmm_b200_dist_chunks": (i32, [i64, i64, i64, u64, i32, i32, C.c_uint, i64, C.POINTER(C.c_int),
                                        _i64p, _i64p]),
        "fpmm_b200_dist_mw_product_device": (i32, [vp, i64, vp, i64, vp, i64, vp, i64, i64, i64, i64,
                                                   u64, i32, i32, u64, i32, vp, C.c_uint,
                                                   C.POINTER(Timing)]),
        "fpmm_b200_random_residues_device": (i32, [vp, i64, i64, i64, i64, u64, u64, i32, vp]),
        "fpmm_b200_verify_device": (i32, [vp, i64, vp, i64, vp, i64, i64, i64, i64, u64, u64, i32, i32,
                                          i32, vp, _i64p]),
        "fpmm_b200_fp64_peak": (i32, [i32, i32, C.POINTER(C.c_double)]),
        "fpmm_b200_i8_peak": (i32, [i32, i32, C.POINTER(C.c_double)]),
        "fpmm_b200_prepare_a_device": (i32, [vp, i64, i64, i64, u64, i32, i32, C.c_uint, i32, vp,
                                             C.POINTER(vp)]),
        "fpmm_b200_mw_product_prepared_device": (i32, [vp, vp, i64, vp, i64, i64, u64, vp, C.c_uint,
                                                       C.POINTER(Timing)]),
        "fpmm_b200_prepared_free": (i32, [vp]),
        "fpmm_b200_finalize": (i32, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(status: int) -> None:
    if status != 0:
        msg = lib().fpmm_b200_last_error().decode(errors="replace")
        raise _ERRS.get(status, Error)(msg)


def _f64(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise Error("matrices must be 2-D")
    if not a.flags.c_contiguous and not (a.strides[1] == 8 and a.strides[0] % 8 == 0):
        a = np.ascontiguousarray(a)
    return a


def _ld(a: np.ndarray) -> int:
    return a.strides[0] // 8 if a.shape[0] > 1 else max(a.shape[1], 1)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


# ------------------------------------------------------------- field / rule
def is_prime_u64(n: int) -> bool:
    """primality.hpp:8 (deterministic Miller-Rabin)."""
    return bool(lib().fpmm_b200_is_prime(n))


def prev_prime(limit: int) -> int:
    """primality.hpp:11: largest prime strictly below ``limit`` (0 if none)."""
    return int(lib().fpmm_b200_prev_prime(limit))


def bitsize(n: int) -> int:
    """int_utils.hpp:15."""
    return int(n).bit_length()


@dataclass(frozen=True)
class FpContext:
    """FpContext<double> (fp_context.hpp:29-77): validated modulus and fl(1/p)."""
    p: int
    prime: bool
    t: int = T

    @staticmethod
    def make(p: int, allow_composite: bool = False) -> "FpContext":
        _check(lib().fpmm_b200_context_check(p, int(allow_composite)))
        return FpContext(p=p, prime=is_prime_u64(p))

    @property
    def pf(self) -> float:
        return float(self.p)

    @property
    def q(self) -> float:
        return 1.0 / float(self.p)

    def bits(self) -> int:
        return bitsize(self.p)

    def residue_mul_fp_safe(self) -> bool:
        return 3 * (self.p - 1) ** 2 <= (1 << (self.t - 1)) * self.p


def word_base(p: int, u: int) -> int:
    """multiword.cpp:7-19: smallest a with a^u >= p."""
    out = C.c_uint64()
    _check(lib().fpmm_b200_word_base(p, u, C.byref(out)))
    return out.value


def word_bound(p: int, u: int) -> int:
    """multiword.hpp:16."""
    return p - 1 if u == 1 else word_base(p, u)


def _opt(v: int) -> Optional[int]:
    return None if v == 0 else v


def max_block_size(max_a: int, max_b: int, p: int, t: int = T) -> Optional[int]:
    """block_product.hpp:13-22 (None == std::nullopt)."""
    out = C.c_uint64()
    _check(lib().fpmm_b200_max_block_size(max_a, max_b, p, t, C.byref(out)))
    return _opt(out.value)


def mw_block_size(u: int, v: int, p: int, t: int = T) -> Optional[int]:
    """planner.hpp:29-31."""
    out = C.c_uint64()
    _check(lib().fpmm_b200_mw_block_size(u, v, p, t, C.byref(out)))
    return _opt(out.value)


def variant_bit_limit(u: int, v: int, t: int = T) -> int:
    """planner.cpp:20-28 with the scan starting at b=2 (F1)."""
    out = C.c_int()
    _check(lib().fpmm_b200_variant_bit_limit(u, v, t, C.byref(out)))
    return out.value


@dataclass(frozen=True)
class Variant:
    u: int
    v: int

    def products(self) -> int:
        return self.u * self.v


kVariants = (Variant(1, 1), Variant(1, 2), Variant(1, 3), Variant(1, 4), Variant(2, 2),
             Variant(2, 3))


def variant_admits_bits(var: Variant, bits: int, t: int = T) -> bool:
    """planner.hpp:44-46."""
    return bits <= variant_bit_limit(var.u, var.v, t)


_CONCAT = {0: "none", 1: "a", 2: "b"}


@dataclass
class ProductPlan:
    """planner.hpp:57-65."""
    u: int = 1
    v: int = 1
    lambda_: int = 1
    concat: str = "none"
    predicted_products: int = 1
    predicted_reductions: int = 0
    storage_entries: int = 0

    def variant(self) -> Variant:
        return Variant(self.u, self.v)

    @staticmethod
    def _from(pl: _Plan) -> "ProductPlan":
        return ProductPlan(pl.u, pl.v, pl.lambda_, _CONCAT[pl.concat], pl.predicted_products,
                           pl.predicted_reductions, pl.storage_entries)


def select_variant(bits: int, m: int, k: int, n: int, t: int = T, min_lambda: int = 1,
                   concat_threshold: int = 256) -> ProductPlan:
    """planner.cpp:93-96."""
    pl = _Plan()
    _check(lib().fpmm_b200_select_variant(bits, m, k, n, t, min_lambda, concat_threshold,
                                          C.byref(pl)))
    return ProductPlan._from(pl)


def plan_for_modulus(p: int, m: int, k: int, n: int, t: int = T, min_lambda: int = 1,
                     concat_threshold: int = 256) -> ProductPlan:
    """planner.cpp:98-101: the (u,v) selection rule at an actual modulus."""
    pl = _Plan()
    _check(lib().fpmm_b200_plan_for_modulus(p, m, k, n, t, min_lambda, concat_threshold,
                                            C.byref(pl)))
    return ProductPlan._from(pl)


def finish_plan(plan: ProductPlan, m: int, k: int, n: int) -> ProductPlan:
    """planner.cpp:30-42."""
    pl = _Plan(plan.u, plan.v, plan.lambda_, {"none": 0, "a": 1, "b": 2}[plan.concat], 0, 0, 0)
    _check(lib().fpmm_b200_finish_plan(C.byref(pl), m, k, n))
    return ProductPlan._from(pl)


def kernel_block(p: int, u: int, v: int) -> int:
    """The fused kernel's exact K-block (terms between in-register reductions)."""
    out = C.c_int64()
    _check(lib().fpmm_b200_kernel_block(p, u, v, C.byref(out)))
    return out.value


RNS_MAX_MODULI = 20


def rns_plan(p: int, k: int) -> dict:
    """RNS engine words for residues < p and contraction length k: the byte
    moduli and the constants of the CRT reconstruction kernel (fpmm_b200_rns_plan)."""
    n = C.c_int()
    mods = (C.c_uint32 * RNS_MAX_MODULI)()
    y = (C.c_uint32 * RNS_MAX_MODULI)()
    g = (C.c_uint32 * RNS_MAX_MODULI)()
    W = (C.c_uint64 * RNS_MAX_MODULI)()
    Mp = C.c_uint64()
    _check(lib().fpmm_b200_rns_plan(p, k, C.byref(n), mods, y, g, W, C.byref(Mp)))
    c = n.value
    return {"n": c, "moduli": list(mods[:c]), "y": list(y[:c]), "g": list(g[:c]), "W": list(W[:c]),
            "Mp": Mp.value}


def select_engine(m: int, k: int, n: int, p: int) -> str:
    """The engine the library default runs for this product shape: "i8" or "rns"."""
    out = C.c_uint()
    _check(lib().fpmm_b200_select_engine(m, k, n, p, C.byref(out)))
    return "rns" if out.value == ENGINE_RNS else "i8"


# ------------------------------------------------------------ synthetic inputs
def mix_seed(a: int, b: int) -> int:
    """mat.hpp:104-110."""
    return int(lib().fpmm_b200_mix_seed(a, b))


def matrix_seed(seed: int, bits: int, m: int, k: int, n: int, which: int) -> int:
    """driver.cpp:14-20."""
    return int(lib().fpmm_b200_matrix_seed(seed, bits, m, k, n, which))


def random_mat(rows: int, cols: int, p: int, seed: int) -> np.ndarray:
    """mat.hpp:112-120: uniform residues in [0,p) from std::mt19937_64(seed)."""
    out = np.empty((rows, cols), dtype=np.float64)
    _check(lib().fpmm_b200_random_mat(rows, cols, p, seed, _ptr(out)))
    return out


# ----------------------------------------------------------------- products
@dataclass
class WordDecomposition:
    """multiword.hpp:19-24: M = sum_i base^i words[i]."""
    base: int
    words: List[np.ndarray] = field(default_factory=list)

    def word_count(self) -> int:
        return len(self.words)


def decompose(M, u: int, F: FpContext) -> WordDecomposition:
    """multiword.hpp:29-54 on the GPU; words bit-identical to the reference's."""
    M = _f64(M)
    rows, cols = M.shape
    words = np.empty((u, rows, cols), dtype=np.float64)
    base = C.c_uint64()
    _check(lib().fpmm_b200_decompose(_ptr(M), _ld(M), rows, cols, F.p, u, _ptr(words),
                                     rows * cols, C.byref(base)))
    return WordDecomposition(base.value, [words[i] for i in range(u)])


def _product(A, B, u, v, lam, F, variant, ngpus=1, flags=0, timing=None, out=None) -> np.ndarray:
    A = _f64(A)
    B = _f64(B)
    if A.shape[1] != B.shape[0]:
        raise Error("multiword product: dimension mismatch")
    m, k = A.shape
    n = B.shape[1]
    if out is not None:
        if out.shape != (m, n) or out.dtype != np.float64 or not out.flags.c_contiguous:
            raise Error("out must be a C-contiguous float64 (m, n) array")
        Cm = out
    else:
        Cm = np.empty((m, n), dtype=np.float64)
    if not F.prime:
        flags |= ALLOW_COMPOSITE
    tm = timing if timing is not None else None
    _check(lib().fpmm_b200_mw_product(_ptr(A), _ld(A), _ptr(B), _ld(B), _ptr(Cm), max(n, 1), m, k,
                                      n, F.p, u, v, lam, variant, ngpus, _eng(flags),
                                      C.byref(tm) if tm is not None else None))
    return Cm


def mw_product(A, B, u: int, v: int, lambda_: int, F: FpContext, kernel=None, *, ngpus: int = 1,
               flags: int = 0, timing: Optional[Timing] = None, out=None) -> np.ndarray:
    """multiword.hpp:133-139: C = A B mod p via the (u,v)-multiword product.

    ``kernel`` is accepted for signature parity (the fused sm_100a kernel is
    always used); ``ngpus`` row-shards C over devices 0..ngpus-1; ``out``
    (e.g. a pinned-memory array) receives C."""
    return _product(A, B, u, v, lambda_, F, PLAIN, ngpus, flags, timing, out)


def mw_product_workspace(A, B, u, v, lambda_, F, kernel=None, **kw) -> np.ndarray:
    """multiword.hpp:248-254 (inverse-free; the composite-modulus variant)."""
    return _product(A, B, u, v, lambda_, F, WORKSPACE, kw.get("ngpus", 1), kw.get("flags", 0),
                    kw.get("timing"))


def mw_product_concat(A, B, u, v, lambda_, F, kernel=None, side="auto", **kw) -> np.ndarray:
    """multiword.hpp:211-218 (same value; every word pair is already one fused tile)."""
    return _product(A, B, u, v, lambda_, F, CONCAT, kw.get("ngpus", 1), kw.get("flags", 0),
                    kw.get("timing"))


def _words_product(da: WordDecomposition, db: WordDecomposition, m, k, n, lam, F, variant,
                   flags=0, timing=None):
    u, v = da.word_count(), db.word_count()
    if u < 1 or v < 1:
        raise Error("multiword product: word counts must be positive")
    aw = np.ascontiguousarray(np.stack([_f64(w) for w in da.words]))
    bw = np.ascontiguousarray(np.stack([_f64(w) for w in db.words]))
    if aw.shape[1:] != (m, k) or bw.shape[1:] != (k, n):
        raise Error("multiword product: dimension mismatch")
    Cm = np.empty((m, n), dtype=np.float64)
    if not F.prime:
        flags |= ALLOW_COMPOSITE
    _check(lib().fpmm_b200_mw_product_words(
        _ptr(aw), m * k, max(k, 1), da.base, u, _ptr(bw), k * n, max(n, 1), db.base, v, _ptr(Cm),
        max(n, 1), m, k, n, F.p, lam, variant, _eng(flags),
        C.byref(timing) if timing is not None else None))
    return Cm


def mw_product_words(da, db, m, k, n, lambda_, F, kernel=None, **kw):
    """multiword.hpp:113-131."""
    return _words_product(da, db, m, k, n, lambda_, F, PLAIN, kw.get("flags", 0), kw.get("timing"))


def mw_product_workspace_words(da, db, m, k, n, lambda_, F, kernel=None, **kw):
    """multiword.hpp:222-246."""
    return _words_product(da, db, m, k, n, lambda_, F, WORKSPACE, kw.get("flags", 0),
                          kw.get("timing"))


def mw_product_concat_words(da, db, m, k, n, lambda_, F, kernel=None, side="auto", **kw):
    """multiword.hpp:155-209."""
    return _words_product(da, db, m, k, n, lambda_, F, CONCAT, kw.get("flags", 0), kw.get("timing"))


def block_gemm_mod(Cm: np.ndarray, A, B, lambda_: int, F: FpContext, kernel=None, *, flags: int = 0) -> None:
    """block_product.hpp:62-73: C <- C + A B mod p in place (C reduced mod p).

    Operands may exceed p (e.g. words bounded by alpha): the value is the
    reference's wherever its panel loop is exact.  CHECK_INPUTS enforces the
    reference's contract (lambda max(A) max(B) + p - 1 <= 2^t, C reduced)."""
    A = _f64(A)
    B = _f64(B)
    if A.shape[0] != Cm.shape[0] or B.shape[1] != Cm.shape[1] or A.shape[1] != B.shape[0]:
        raise Error("block_gemm_mod: dimension mismatch")
    if Cm.dtype != np.float64 or not Cm.flags.c_contiguous:
        raise Error("block_gemm_mod: C must be a C-contiguous float64 matrix")
    m, k = A.shape
    n = B.shape[1]
    _check(lib().fpmm_b200_block_gemm_mod(_ptr(Cm), max(n, 1), _ptr(A), _ld(A), _ptr(B), _ld(B), m,
                                          k, n, lambda_, F.p, _eng(flags)))


class GemmKernel:
    """GemmKernel<double> (gemm_kernel.hpp:13-19): exact C += A B on panels."""

    def accumulate(self, c: np.ndarray, a, b) -> None:
        a = _f64(a)
        b = _f64(b)
        if c.dtype != np.float64 or c.strides[1] != 8:
            raise Error("accumulate: C must be a row-major float64 view")
        m, w = a.shape
        n = b.shape[1]
        if c.shape != (m, n) or b.shape[0] != w:
            raise Error("accumulate: dimension mismatch")
        _check(lib().fpmm_b200_accumulate(c.ctypes.data_as(_dp), _ld(c), _ptr(a), _ld(a), _ptr(b),
                                          _ld(b), m, w, n))

    def name(self) -> str:
        return "b200"


_B200 = GemmKernel()


def b200_kernel() -> GemmKernel:
    return _B200


def kernel_by_name(name: str) -> Optional[GemmKernel]:
    """gemm_kernel.hpp:57-62, with the B200 kernel registered as "b200"."""
    return _B200 if name in ("b200", "accelerated") else None


# ----------------------------------------------------------- device tensors
CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy


def _stream_handle(stream, device=None):
    """ctypes value for a torch stream.  None -> torch's current stream on
    `device`, so a call on torch tensors is ordered after the torch work that
    produced them (e.g. a non_blocking H2D copy) and before the work that
    reads its result; the default (legacy) stream, whose handle is 0, ->
    cudaStreamLegacy."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream or CUDA_STREAM_LEGACY


def _dev_ld(t) -> int:
    if t.dim() != 2 or t.stride(1) != 1:
        raise Error("device matrices must be 2-D row-major (stride(1) == 1)")
    return t.stride(0) if t.shape[0] > 1 else max(t.shape[1], 1)


def mw_product_device(A, B, Cout, p: int, u: int, v: int, lambda_: int, *, variant: int = PLAIN,
                      flags: int = 0, stream=None, timing: Optional[Timing] = None,
                      allow_composite: bool = False) -> None:
    """C = A B mod p on device-resident torch float64 tensors (same device)."""
    m, k = A.shape
    n = B.shape[1]
    if B.shape[0] != k or tuple(Cout.shape) != (m, n):
        raise Error("multiword product: dimension mismatch")
    if allow_composite:
        flags |= ALLOW_COMPOSITE
    dev = A.device.index
    sp = _stream_handle(stream, dev)
    _check(lib().fpmm_b200_mw_product_device(A.data_ptr(), _dev_ld(A), B.data_ptr(), _dev_ld(B),
                                             Cout.data_ptr(), _dev_ld(Cout), m, k, n, p, u, v,
                                             lambda_, variant, dev, sp, _eng(flags),
                                             C.byref(timing) if timing is not None else None))


class PreparedA:
    """A's words packed once and kept resident in HBM (the reference's
    unbalanced scenario decomposes A outside the timer, driver.cpp:215-218)."""

    def __init__(self, A, p: int, u: int, v: int, *, flags: int = 0, stream=None,
                 allow_composite: bool = False):
        if allow_composite:
            flags |= ALLOW_COMPOSITE
        self.m, self.k = A.shape
        self.p, self.u, self.v = p, u, v
        self.device = A.device.index
        h = C.c_void_p()
        _check(lib().fpmm_b200_prepare_a_device(A.data_ptr(), _dev_ld(A), self.m, self.k, p, u, v,
                                                _eng(flags), self.device, _stream_handle(stream, self.device),
                                                C.byref(h)))
        self._h = h

    def product(self, B, Cout, lambda_: int, *, flags: int = 0, stream=None,
                timing: Optional[Timing] = None) -> None:
        """Cout (m x n) = A B mod p (device tensors)."""
        n = B.shape[1]
        if B.shape[0] != self.k or tuple(Cout.shape) != (self.m, n):
            raise Error("multiword product: dimension mismatch")
        _check(lib().fpmm_b200_mw_product_prepared_device(
            self._h, B.data_ptr(), _dev_ld(B), Cout.data_ptr(), _dev_ld(Cout), n, lambda_,
            _stream_handle(stream, self.device), flags, C.byref(timing) if timing is not None else None))

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            _check(lib().fpmm_b200_prepared_free(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def decompose_device(M, p: int, u: int, words, stream=None) -> int:
    """Reference-identical words of device matrix M into words (u x rows x cols)."""
    rows, cols = M.shape
    base = C.c_uint64()
    sp = _stream_handle(stream, M.device.index)
    _check(lib().fpmm_b200_decompose_device(M.data_ptr(), _dev_ld(M), rows, cols, p, u,
                                            words.data_ptr(), rows * cols, C.byref(base),
                                            M.device.index, sp))
    return base.value


def accumulate_device(Cm, A, B, stream=None) -> None:
    m, w = A.shape
    n = B.shape[1]
    sp = _stream_handle(stream, A.device.index)
    _check(lib().fpmm_b200_accumulate_device(Cm.data_ptr(), _dev_ld(Cm), A.data_ptr(), _dev_ld(A),
                                             B.data_ptr(), _dev_ld(B), m, w, n, A.device.index, sp))


def random_residues_device(M, p: int, seed: int, row0: int = 0, stream=None) -> None:
    """Fill device tensor M (rows row0.. of a global matrix) with uniform residues in [0,p)."""
    rows, cols = M.shape
    sp = _stream_handle(stream, M.device.index)
    _check(lib().fpmm_b200_random_residues_device(M.data_ptr(), _dev_ld(M), rows, cols, row0, p,
                                                  seed, M.device.index, sp))


def verify_device(A, B, Cm, p: int, *, seed: int = 1, trials: int = 2, samples: int = 64,
                  stream=None) -> dict:
    """Exact on-device check of C = A B mod p (device tensors): C's range,
    Freivalds trials A (B s) == C s mod p, sampled exact entries
    (fpmm_b200_verify_device).  ``ok`` is True when every count is zero."""
    m, k = A.shape
    n = B.shape[1]
    if B.shape[0] != k or tuple(Cm.shape) != (m, n):
        raise Error("verify: dimension mismatch")
    out = (C.c_int64 * 5)()
    _check(lib().fpmm_b200_verify_device(A.data_ptr(), _dev_ld(A), B.data_ptr(), _dev_ld(B), Cm.data_ptr(),
                                         _dev_ld(Cm), m, k, n, p, seed, trials, samples, A.device.index,
                                         _stream_handle(stream, A.device.index), out))
    r = {"range": out[0], "freivalds_rows": out[1], "samples_bad": out[2], "first_bad": (out[3], out[4]),
         "trials": trials, "samples": samples}
    r["ok"] = out[0] == 0 and out[1] == 0 and out[2] == 0
    return r


def i8_peak(device: int = 0, iters: int = 200000) -> float:
    """Measured int8 tensor-core (tcgen05 kind::i8) peak of `device` in TOP/s."""
    out = C.c_double()
    _check(lib().fpmm_b200_i8_peak(device, iters, C.byref(out)))
    return out.value


def fp64_peak(device: int = 0, iters: int = 20000) -> float:
    """Measured FP64 tensor-pipe (DMMA) peak of `device` in TFLOP/s."""
    out = C.c_double()
    _check(lib().fpmm_b200_fp64_peak(device, iters, C.byref(out)))
    return out.value


def device_count() -> int:
    out = C.c_int()
    _check(lib().fpmm_b200_device_count(C.byref(out)))
    return out.value


def finalize() -> None:
    _check(lib().fpmm_b200_finalize())
