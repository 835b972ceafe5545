"""compute-sanitizer workload for rns_tile_kernel (FPMM_B200_RNS_TILE=1 forced):
small ragged shapes with shared-memory and TMEM residue planes, against the u128 oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["FPMM_B200_RNS_TILE"] = "1"
import oracle as O  # noqa: E402
import paper_2601_07508_b200 as F  # noqa: E402

for bits, (m, k, n) in ((52, (300, 200, 130)), (20, (64, 100, 33)), (40, (257, 129, 300)), (12, (513, 64, 140))):
    p, A, B = O.seeded_inputs(m, k, n, bits)
    pl = F.plan_for_modulus(p, m, k, n)
    C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), flags=F.ENGINE_RNS)
    assert (C == O.exact_mod_gemm(A, B, p)).all(), bits
print("sanitize tile workload ok")
