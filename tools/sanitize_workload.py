import sys; sys.path.insert(0, '.')
import numpy as np, oracle as O, paper_2601_07508_b200 as F
for eng in (F.ENGINE_DMMA, F.ENGINE_I8, F.ENGINE_RNS):
    for bits, (m, k, n) in ((52, (130, 200, 70)), (20, (64, 100, 33)), (40, (300, 129, 257))):
        p, A, B = O.seeded_inputs(m, k, n, bits)
        pl = F.plan_for_modulus(p, m, k, n)
        C = F.mw_product(A, B, pl.u, pl.v, pl.lambda_, F.FpContext.make(p), flags=eng)
        assert (C == O.exact_mod_gemm(A, B, p)).all()
print("sanitize workload ok")
