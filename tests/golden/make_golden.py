"""Generate tests/golden/golden.json by running the REFERENCE library itself.

The reference (/root/reference/proj/src, unmodified) is compiled by
oracle/Makefile into oracle/_ref/libfpmm_ref.so; this script drives its own
mw_product / mw_product_workspace / mw_product_concat / decompose / planner on
the reference driver's seeded inputs (driver.cpp:14-20, mat.hpp:112-120) and
records the outputs.  Run here (needs /root/reference):

    python tests/golden/make_golden.py

The JSON is committed; the GPU box never needs /root/reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

VARIANTS = [(1, 1), (1, 2), (1, 3), (1, 4), (2, 2), (2, 3)]
BITS = [5, 20, 26, 30, 35, 39, 42, 48, 52]          # SPEC.md acceptance 1
DIMS = [(17, 33, 9), (64, 64, 64), (128, 300, 32)]  # SPEC.md acceptance 1


def ref_lambda(u, v, p, k):
    R = O.ref()
    out = O.C.c_uint64()
    assert R.ref_mw_block_size(u, v, p, 53, O.C.byref(out)) == 0
    return min(out.value, k) if out.value else 0


def main():
    R = O.ref()
    assert R is not None, "reference library not built (make -C oracle)"
    cases = []
    for (m, k, n) in DIMS:
        for bits in BITS:
            p = int(R.ref_prev_prime(1 << bits))
            A = np.empty((m, k)); B = np.empty((k, n))
            R.ref_random_mat(m, k, p, R.ref_matrix_seed(1, bits, m, k, n, 0xA), O._ptr(A))
            R.ref_random_mat(k, n, p, R.ref_matrix_seed(1, bits, m, k, n, 0xB), O._ptr(B))
            for (u, v) in VARIANTS:
                if bits > O.variant_bit_limit(u, v):
                    continue
                lam = ref_lambda(u, v, p, k)
                if lam == 0:
                    continue
                C0 = O.ref_mw_product(A, B, p, u, v, lam, variant=0, accelerated=False)
                C1 = O.ref_mw_product(A, B, p, u, v, lam, variant=1, accelerated=False)
                C2 = O.ref_mw_product(A, B, p, u, v, lam, variant=2, accelerated=False)
                assert (C0 == C1).all() and (C0 == C2).all()
                case = dict(m=m, k=k, n=n, bits=bits, p=p, u=u, v=v, lam=lam, seed=1,
                            A00=int(A[0, 0]), B00=int(B[0, 0]), C00=int(C0[0, 0]),
                            Clast=int(C0[-1, -1]), fnv1a64=O.fnv1a64(C0))
                if m * n <= 200:
                    case["C"] = [int(x) for x in C0.ravel()]
                cases.append(case)
    # SURVEY.md Appendix B shapes (C corner values are quoted there)
    for (m, k, n, bits, u, v) in [(64, 64, 64, 50, 2, 2), (16, 262144, 16, 48, 2, 2),
                                  (128, 256, 128, 40, 2, 2), (128, 128, 128, 52, 2, 2),
                                  (128, 128, 128, 45, 2, 2), (128, 128, 128, 39, 1, 3),
                                  (128, 128, 128, 35, 1, 2), (128, 128, 128, 26, 1, 1),
                                  (128, 128, 128, 20, 1, 1), (1024, 1024, 1024, 50, 2, 2)]:
        p = int(R.ref_prev_prime(1 << bits))
        A = np.empty((m, k)); B = np.empty((k, n))
        R.ref_random_mat(m, k, p, R.ref_matrix_seed(1, bits, m, k, n, 0xA), O._ptr(A))
        R.ref_random_mat(k, n, p, R.ref_matrix_seed(1, bits, m, k, n, 0xB), O._ptr(B))
        lam = ref_lambda(u, v, p, k)
        C0 = O.ref_mw_product(A, B, p, u, v, lam, variant=0, accelerated=True)
        cases.append(dict(m=m, k=k, n=n, bits=bits, p=p, u=u, v=v, lam=lam, seed=1,
                          A00=int(A[0, 0]), B00=int(B[0, 0]), C00=int(C0[0, 0]),
                          Clast=int(C0[-1, -1]), fnv1a64=O.fnv1a64(C0), appendix_b=True))
    # reference decompose words (multiword.hpp:29-54) on a few matrices
    decomp = []
    for bits, u in [(37, 3), (38, 3), (40, 2), (45, 2), (47, 2), (51, 2), (52, 4)]:
        p = int(R.ref_prev_prime(1 << bits))
        M = np.empty((8, 16))
        R.ref_random_mat(8, 16, p, 1000 + bits, O._ptr(M))
        M[0, :4] = [0, p - 1, 1, p // 2]
        W = np.empty((u, 8, 16)); base = O.C.c_uint64()
        assert R.ref_decompose(O._ptr(M), 8, 16, p, u, O._ptr(W), O.C.byref(base)) == 0
        decomp.append(dict(bits=bits, p=p, u=u, base=base.value, M=[int(x) for x in M.ravel()],
                           words=[[int(x) for x in W[i].ravel()] for i in range(u)]))
    out = dict(generator="tests/golden/make_golden.py (reference library oracle/_ref)",
               hash="fnv1a64 over the 8 little-endian bytes of each C value as u64, row-major",
               cases=cases, decompose=decomp)
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0)
    print("wrote", path, len(cases), "cases")


if __name__ == "__main__":
    main()
