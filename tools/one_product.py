"""Run one device-resident product (for ncu captures): python tools/one_product.py BITS [M K N] [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07508_b200 as F  # noqa: E402

bits = int(sys.argv[1])
m, k, n = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (8192, 8192, 8192)
reps = int(sys.argv[5]) if len(sys.argv) >= 6 else 2
p = F.prev_prime(1 << bits)
pl = F.plan_for_modulus(p, m, k, n)
A = torch.empty((m, k), dtype=torch.float64, device="cuda")
B = torch.empty((k, n), dtype=torch.float64, device="cuda")
C = torch.empty((m, n), dtype=torch.float64, device="cuda")
F.random_residues_device(A, p, 1)
F.random_residues_device(B, p, 2)
for _ in range(reps):
    tm = F.Timing()
    eng = {'i8': F.ENGINE_I8, 'dmma': F.ENGINE_DMMA, 'rns': F.ENGINE_RNS}[os.environ.get('ENGINE', 'dmma')]
    F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, timing=tm, flags=eng)
    print(bits, (pl.u, pl.v, pl.lambda_), tm.as_dict(),
          "eff %.1f GF/s, fp64 %.2f TF/s" % (2 * m * k * n / tm.gemm_ms / 1e6, 2 * pl.u * pl.v * m * k * n / tm.gemm_ms / 1e9))
