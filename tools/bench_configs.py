"""Measure every BASELINE.json config once per engine (device-resident inputs).

  python tools/bench_configs.py [--out profiles/round1/configs.json] [--only c3,c5]

configs[0] 1024^3 / 50-bit; configs[1] the 8192^3 sweep is bench.py's default
workload; configs[2] 32768^3 / 52-bit (1 GPU here); configs[3] 4096 x 262144
x 4096 / 48-bit; configs[4] 65536 x 256 x 65536 / 40-bit (rule picks (2,2)).
Plus the paper's unbalanced preset 10923 x 32768 x 32 with A's words prepared
outside the timer (driver.cpp:215-218).  Each point: 1 warm-up + R timed runs,
CUDA events on one stream, inputs larger than L2.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2601_07508_b200 as F  # noqa: E402

CONFIGS = {
    "c1": (1024, 1024, 1024, 50, 20),
    "c3": (32768, 32768, 32768, 52, 1),
    "c4": (4096, 262144, 4096, 48, 2),
    "c5": (65536, 256, 65536, 40, 3),
    "unbalanced": (10923, 32768, 32, 48, 20),
}


def run(name, engine, stream):
    m, k, n, bits, runs = CONFIGS[name]
    p = F.prev_prime(1 << bits)
    pl = F.plan_for_modulus(p, m, k, n)
    A = torch.empty((m, k), dtype=torch.float64, device="cuda")
    B = torch.empty((k, n), dtype=torch.float64, device="cuda")
    C = torch.empty((m, n), dtype=torch.float64, device="cuda")
    F.random_residues_device(A, p, F.matrix_seed(1, bits, m, k, n, 0xA))
    F.random_residues_device(B, p, F.matrix_seed(1, bits, m, k, n, 0xB))
    fl = {"i8": F.ENGINE_I8, "rns": F.ENGINE_RNS, "dmma": F.ENGINE_DMMA, "auto": 0}[engine]
    pa = F.PreparedA(A, p, pl.u, pl.v, flags=fl) if name == "unbalanced" else None

    def once(tm=None):
        if pa is None:
            F.mw_product_device(A, B, C, p, pl.u, pl.v, pl.lambda_, flags=fl | F.ASYNC, stream=stream, timing=tm)
        else:
            pa.product(B, C, pl.lambda_, flags=F.ASYNC, stream=stream, timing=tm)

    once()
    torch.cuda.synchronize()
    # let the power-capped clock recover from the previous measurement (a slow
    # engine's long run left the next one up to 20% low)
    import time
    time.sleep(2.0)
    once()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(runs):
        once()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / runs
    tm = F.Timing()
    once(tm)
    torch.cuda.synchronize()
    if pa is not None:
        pa.close()
    del A, B, C
    torch.cuda.empty_cache()
    return {"m": m, "k": k, "n": n, "bits": bits, "p": p, "u": pl.u, "v": pl.v, "lambda": pl.lambda_,
            "engine": engine, "ms": round(ms, 3), "eff_gflops": round(2.0 * m * k * n / ms / 1e6, 1),
            "gemm_ms": round(tm.gemm_ms, 3), "pack_ms": round(tm.pack_ms, 3), "lambda_k": tm.lambda_k,
            "runs": runs, "a_prepared_outside_timer": name == "unbalanced"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=",".join(CONFIGS))
    ap.add_argument("--engines", default="auto,rns,i8,dmma")
    args = ap.parse_args()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    res = []
    for name in args.only.split(","):
        for eng in args.engines.split(","):
            r = run(name, eng, stream)
            r["config"] = name
            print(json.dumps(r), flush=True)
            res.append(r)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
