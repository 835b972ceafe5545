"""Breakdown of one host-buffer product (the bench's e2e path): python tools/e2e_probe.py BITS [N]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07508_b200 as F  # noqa: E402

bits = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
p = F.prev_prime(1 << bits)
pl = F.plan_for_modulus(p, n, n, n)
pin = lambda: torch.empty((n, n), dtype=torch.float64, pin_memory=True)  # noqa: E731
hA, hB, hC = pin(), pin(), pin()
dA = torch.empty((n, n), dtype=torch.float64, device="cuda")
F.random_residues_device(dA, p, 1)
hA.copy_(dA)
F.random_residues_device(dA, p, 2)
hB.copy_(dA)
torch.cuda.synchronize()
t = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t[0].record()
x = dA.cpu()
t[1].record()
torch.cuda.synchronize()
print("torch D2H pageable %.2f GB/s" % (8 * n * n / t[0].elapsed_time(t[1]) / 1e6))
d = torch.empty((n, n), dtype=torch.float64, device="cuda")
t[0].record()
d.copy_(hA, non_blocking=True)
t[1].record()
torch.cuda.synchronize()
print("pinned H2D %.2f GB/s" % (8 * n * n / t[0].elapsed_time(t[1]) / 1e6))
for r in range(3):
    tm = F.Timing()
    t0 = time.perf_counter()
    F.mw_product(hA.numpy(), hB.numpy(), pl.u, pl.v, pl.lambda_, F.FpContext.make(p), out=hC.numpy(), timing=tm)
    dt = time.perf_counter() - t0
    print("wall %.2f ms" % (dt * 1e3), {k: round(v, 3) if isinstance(v, float) else v for k, v in tm.as_dict().items()})

# sweep mode (as bench.py's e2e leg): per-bitsize wall time with and without
# refreshing the pinned inputs from the device between calls
if len(sys.argv) > 3 and sys.argv[3] == "sweep":
    for refresh in (False, True):
        tot = 0.0
        per = []
        for b in range(20, 53):
            p = F.prev_prime(1 << b)
            pl = F.plan_for_modulus(p, n, n, n)
            if refresh:
                F.random_residues_device(dA, p, b)
                hA.copy_(dA)
                hB.copy_(dA)
            else:
                F.random_residues_device(d, p, b)  # keep the inputs valid residues for p
                hA.copy_(d)
                hB.copy_(d)
            torch.cuda.synchronize()
            tm = F.Timing()
            t0 = time.perf_counter()
            F.mw_product(hA.numpy(), hB.numpy(), pl.u, pl.v, pl.lambda_, F.FpContext.make(p), out=hC.numpy(),
                         timing=tm)
            dt = time.perf_counter() - t0
            tot += dt
            per.append((b, round(dt * 1e3, 2), round(tm.h2d_ms, 2), round(tm.gemm_ms, 2), round(tm.total_ms, 2)))
        print("refresh" if refresh else "plain", "sweep %.1f ms" % (tot * 1e3), per)
