"""A/B of the FP64 engine's in-register reductions at 8192^3 (device-resident):
the one-DFMA form (default where cheaper) against the 3-instruction form
(FPMM_B200_CLASSIC_REDUCE=1), per bitsize, with a bitwise comparison of C.

  python tools/dmma_ab.py [BITS,...] [M K N] [REPS]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07508_b200 as F  # noqa: E402

bits_list = [int(b) for b in (sys.argv[1] if len(sys.argv) > 1 else "34,35,39,40,44,48,50,51,52").split(",")]
m, k, n = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (8192, 8192, 8192)
reps = int(sys.argv[5]) if len(sys.argv) >= 6 else 3
PEAK = 37.07e12
A = torch.empty((m, k), dtype=torch.float64, device="cuda")
B = torch.empty((k, n), dtype=torch.float64, device="cuda")
C0 = torch.empty((m, n), dtype=torch.float64, device="cuda")
C1 = torch.empty((m, n), dtype=torch.float64, device="cuda")
rows = []
for bits in bits_list:
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, m, k, n)
    F.random_residues_device(A, p, 1 + bits)
    F.random_residues_device(B, p, 2 + bits)
    res = {}
    for mode, C in (("classic", C0), ("fast", C1)):
        if mode == "classic":
            os.environ["FPMM_B200_CLASSIC_REDUCE"] = "1"
        else:
            os.environ.pop("FPMM_B200_CLASSIC_REDUCE", None)
        best = None
        for _ in range(reps):
            tm = F.Timing()
            F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, timing=tm, flags=F.ENGINE_DMMA)
            best = tm if best is None or tm.gemm_ms < best.gemm_ms else best
        res[mode] = {"gemm_ms": round(best.gemm_ms, 3), "lambda_k": best.lambda_k, "words": best.words,
                     "eff_tf": round(2 * m * k * n / best.gemm_ms / 1e9, 2),
                     "uv_frac": round(2 * pl.u * pl.v * m * k * n / (best.gemm_ms * 1e-3) / PEAK, 4)}
    torch.cuda.synchronize()
    same = bool(torch.equal(C0, C1))
    row = {"bits": bits, "rule_uv": [pl.u, pl.v], "lambda": pl.lambda_, **res, "bitwise_equal": same}
    rows.append(row)
    print(json.dumps(row), flush=True)
os.environ.pop("FPMM_B200_CLASSIC_REDUCE", None)
if not all(r["bitwise_equal"] for r in rows):
    sys.exit("classic and fast reductions disagree")
