"""rns_tile_kernel (on-chip CRT) against the parked-residue RNS path: C bit-identical
between FPMM_B200_RNS_TILE=0 and =1, the device verifier on the tile result, the
oracle on small shapes, and per-mode timing.  python tools/tile_check.py [quick|short|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2601_07508_b200 as F  # noqa: E402

SMALL = [(256, 64, 128, 20), (512, 256, 512, 40), (1000, 300, 700, 52), (300, 17, 260, 12), (777, 129, 1025, 31),
         (256, 256, 256, 5), (513, 512, 385, 48), (2048, 1024, 2048, 36)]
BIG = [(16384, 256, 16384, 20), (16384, 256, 16384, 30), (16384, 256, 16384, 40), (16384, 256, 16384, 52),
       (8192, 512, 8192, 40), (8192, 1024, 8192, 40), (8192, 2048, 8192, 40), (8192, 4096, 8192, 40),
       (8192, 8192, 8192, 20), (8192, 8192, 8192, 40), (8192, 8192, 8192, 52), (65536, 256, 65536, 40)]


def product(A, B, C, p, reps=0):
    fl = F.ENGINE_RNS | F.ASYNC
    pl = F.plan_for_modulus(p, A.shape[0], A.shape[1], B.shape[1])
    uvl = (pl.u, pl.v, pl.lambda_)
    F.mw_product_device(A, B, C, p, *uvl, flags=fl)
    torch.cuda.synchronize()
    if not reps:
        return None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        F.mw_product_device(A, B, C, p, *uvl, flags=fl)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


SHORT = [(16384, 256, 16384, 20), (16384, 256, 16384, 40), (16384, 256, 16384, 52), (8192, 512, 8192, 40),
         (65536, 256, 65536, 40)]


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    shapes = {"quick": SMALL, "short": SMALL[:3] + SHORT, "all": SMALL + BIG}[which]
    import oracle as O
    bad = 0
    for (m, k, n, bits) in shapes:
        p = F.prev_prime(1 << bits)
        A = torch.empty((m, k), dtype=torch.float64, device="cuda")
        B = torch.empty((k, n), dtype=torch.float64, device="cuda")
        F.random_residues_device(A, p, 11)
        F.random_residues_device(B, p, 12)
        if m * n <= 1 << 22:  # worst case on one corner: all p-1
            A[:7, :] = p - 1
            B[:, :5] = p - 1
        Cs, ms = {}, {}
        for mode in ("0", "1"):
            os.environ["FPMM_B200_RNS_TILE"] = mode
            Cs[mode] = torch.full((m, n), -1.0, dtype=torch.float64, device="cuda")
            ms[mode] = product(A, B, Cs[mode], p, reps=0 if m * n * k < 1 << 30 else 3)
        same = torch.equal(Cs["0"], Cs["1"])
        ok = same
        extra = ""
        if m * n * k <= 1 << 28:
            want = O.exact_mod_gemm(A.cpu().numpy(), B.cpu().numpy(), p)
            ok = ok and np.array_equal(Cs["1"].cpu().numpy(), want)
            extra = " oracle"
        else:
            v = F.verify_device(A, B, Cs["1"], p)
            ok = ok and v["ok"]
            extra = " verify %s" % v["ok"]
        bad += not ok
        t = ""
        if ms["0"]:
            t = " parked %.3f ms  tile %.3f ms (%.1f / %.1f TF-eff)" % (
                ms["0"], ms["1"], 2e-9 * m * k * n / ms["0"], 2e-9 * m * k * n / ms["1"])
        print("%6d %6d %6d %2d bits n=%2d: %s same=%s%s%s" % (
            m, k, n, bits, F.rns_plan(p, k)["n"], "OK " if ok else "BAD", same, extra, t), flush=True)
        del A, B, Cs
        torch.cuda.empty_cache()
    print("tile_check: %d bad" % bad)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
