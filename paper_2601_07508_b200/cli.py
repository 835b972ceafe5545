"""Command-line front end mirroring the reference's ``fpmm`` tool
(/root/reference/proj/tools/fpmm_cli.cpp:92-169) for the B200 library:

  python -m paper_2601_07508_b200.cli bench [--scenario square|unbalanced] [--dims m,k,n]
        [--scale S] [--bits 20 26 ...] [--variant u,v|auto ...] [--lambda auto|N]
        [--kernel b200|b200-rns|b200-i8|b200-dmma|b200-dmma-exact] [--runs R] [--seed S] [--out CSV]
        [--extended] [--device-resident]
  python -m paper_2601_07508_b200.cli check [--bits ...] [--dims m,k,n ...] [--variant u,v ...]
        [--op plain|concat|workspace] [--seed S] [--seeds N] [--kernel ...] [--lambda N] [--checked]
        [--trials T] [--dump-dir DIR] [--quiet]
  python -m paper_2601_07508_b200.cli crossover bench.csv [--out CSV]
  python -m paper_2601_07508_b200.cli plan --bits B [--dims m,k,n] [--min-lambda L]

``bench`` writes the reference's CSV schema v1 (bench.cpp:14-16, 35-45); with
``--extended`` it appends engine, lambda_k, gpus and device-time columns.
Timing follows run_bench (driver.cpp:222-243): for the square scenario the
block size, both decompositions and the product are inside the timer; for
the unbalanced scenario A's words are prepared once outside it.  Inputs are
host matrices (the drop-in's calling convention), so the timer also covers
the PCIe transfers.  ``crossover`` reproduces crossover_table
(bench.cpp:93-136).  ``check`` is the oracle-equivalence suite of
run_check (driver.cpp:37-140, defaults driver.hpp:21-33) with PASS/FAIL/SKIP
lines (fpmm_cli.cpp:52-66).  It verifies C without recomputing it on the CPU:
exact Freivalds trials (C s == A (B s) mod p in Python integers) plus sampled
entries, each an exact dot product, which name the first mismatching
position.  ``--checked`` (the reference's shadow replay) turns on
CHECK_EXACTNESS; ``--dump-dir`` writes a failing case's A and B as .npy.  Exit codes follow the reference: 0 ok, 1 failure,
2 usage error (fpmm_cli.cpp:14-16).
"""
from __future__ import annotations

import argparse
import csv
import io
import sys
import time

import numpy as np

from . import (CHECK_EXACTNESS, DMMA_EXACT_WORDS, ENGINE_DMMA, ENGINE_I8, ENGINE_RNS, Error, FpContext, InfeasibleError,
               Timing, kVariants, mw_product, mw_product_concat, mw_product_workspace, variant_bit_limit,
               matrix_seed, mw_block_size, plan_for_modulus, prev_prime, random_mat,
               variant_admits_bits)

SCHEMA_VERSION = 1
HEADER = ["schema_version", "scenario", "m", "k", "n", "bits", "p", "u", "v", "concat", "lambda",
          "kernel", "runs", "t_avg_s", "eff_gflops", "status"]
EXTENDED = ["engine", "lambda_k", "gpus", "device_ms"]
KERNELS = {"b200": 0, "b200-i8": ENGINE_I8, "b200-rns": ENGINE_RNS, "b200-dmma": ENGINE_DMMA,
           # the FP64 engine with exactly the variant's (u,v) words: per-variant timings for crossover
           "b200-dmma-exact": ENGINE_DMMA | DMMA_EXACT_WORDS}


def preset_dims(scenario: str, scale: float):
    """driver.cpp:142-157."""
    def scaled(base, quantum, floor_to):
        q = int(round(base * scale / quantum)) * quantum
        return max(q, floor_to)
    if scenario == "square":
        n = scaled(10016, 32, 32)
        return n, n, n
    if scenario == "unbalanced":
        return max(int(round(10923 * scale)), 1), scaled(32768, 32, 32), 32
    raise Error("unknown scenario '%s' (square|unbalanced)" % scenario)


def parse_dims(s: str):
    parts = [int(x) for x in s.split(",")]
    if len(parts) != 3 or min(parts) < 1:
        raise Error("dims must be m,k,n with positive entries")
    return tuple(parts)


def parse_variants(vs):
    if not vs or vs == ["auto"]:
        return None
    out = []
    for v in vs:
        u, w = (int(x) for x in v.split(","))
        out.append((u, w))
    return out


def effective_gflops(m, k, n, t):
    """bench.cpp:29-33."""
    return 2.0 * m * k * n / t * 1e-9 if t > 0 else 0.0


def run_bench(args) -> list:
    m, k, n = parse_dims(args.dims) if args.dims else preset_dims(args.scenario, args.scale)
    flags = KERNELS[args.kernel]
    variants = parse_variants(args.variant)
    rows = []
    for bits in args.bits:
        p = prev_prime(1 << bits) if bits <= 62 else 0
        var_list = variants or [None]
        for var in var_list:
            rec = dict(schema_version=SCHEMA_VERSION, scenario=args.scenario, m=m, k=k, n=n, bits=bits,
                       p=0, u=1, v=1, concat="none", kernel=args.kernel, runs=args.runs, t_avg_s=0.0,
                       eff_gflops=0.0, status="ok", engine="", lambda_k=0, gpus=1, device_ms=0.0)
            rec["lambda"] = 0
            try:
                if p < 5 or p.bit_length() != bits:
                    raise InfeasibleError("no prime of this bitsize")
                if var is None:
                    pl = plan_for_modulus(p, m, k, n)
                    u, v = pl.u, pl.v
                else:
                    u, v = var
                    if bits > 52 or not variant_admits_bits(type(kVariants[0])(u, v), bits):
                        raise InfeasibleError("variant does not admit this bitsize")
                rec.update(p=p, u=u, v=v)
                F = FpContext.make(p)
                A = random_mat(m, k, p, matrix_seed(args.seed, bits, m, k, n, 0xA))
                B = random_mat(k, n, p, matrix_seed(args.seed, bits, m, k, n, 0xB))
                Cm = np.empty((m, n))
                prepared = None
                dev_in = None
                if args.device_resident and args.scenario == "square":
                    import torch
                    dev_in = (torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(),
                              torch.empty((m, n), dtype=torch.float64, device="cuda"))
                if args.scenario == "unbalanced":
                    import torch
                    from . import PreparedA
                    prepared = PreparedA(torch.from_numpy(A).cuda(), p, u, v, flags=flags)
                    dB = torch.empty((k, n), dtype=torch.float64, device="cuda")
                    dC = torch.empty((m, n), dtype=torch.float64, device="cuda")
                    hB = torch.from_numpy(B).pin_memory()
                    hC = torch.empty((m, n), dtype=torch.float64).pin_memory()
                total = dev = 0.0
                lam_used = 0
                for r in range(args.runs + 1):  # run 0 is an untimed warm-up (allocations)
                    tm = Timing()
                    t0 = time.perf_counter()
                    lam = int(args.lambda_) if args.lambda_ != "auto" else min(mw_block_size(u, v, p) or 0, k)
                    if lam < 1:
                        raise InfeasibleError("block size infeasible")
                    if dev_in is not None:
                        from . import mw_product_device
                        mw_product_device(dev_in[0], dev_in[1], dev_in[2], p, u, v, lam, flags=flags, timing=tm)
                    elif prepared is None:
                        from . import mw_product
                        mw_product(A, B, u, v, lam, F, flags=flags, timing=tm, out=Cm)
                    else:
                        dB.copy_(hB, non_blocking=True)
                        prepared.product(dB, dC, lam, timing=tm)
                        hC.copy_(dC)
                    dt = time.perf_counter() - t0
                    if r > 0:
                        total += dt
                        dev += tm.total_ms
                    lam_used = lam
                rec["lambda"] = lam_used
                # device-resident runs are timed by the library's CUDA events (no PCIe)
                rec["t_avg_s"] = (dev / 1e3 if dev_in is not None else total) / args.runs
                rec["eff_gflops"] = effective_gflops(m, k, n, rec["t_avg_s"])
                rec["engine"] = ("rns" if flags & ENGINE_RNS else "dmma" if flags & ENGINE_DMMA
                                 else "i8" if flags & ENGINE_I8 else "auto")
                rec["lambda_k"] = tm.lambda_k
                rec["device_ms"] = dev / args.runs
                if prepared is not None:
                    prepared.close()
            except InfeasibleError:
                rec["status"] = "infeasible"
            rows.append(rec)
    return rows


def write_csv(rows, out, extended=False):
    cols = HEADER + (EXTENDED if extended else [])
    w = csv.writer(out, lineterminator="\n")
    w.writerow(cols)
    for r in rows:
        vals = []
        for c in cols:
            x = r[c]
            if c == "t_avg_s":
                x = "%.9g" % x
            elif c == "eff_gflops":
                x = "%.6g" % x
            elif c == "device_ms":
                x = "%.6g" % x
            vals.append(x)
        w.writerow(vals)


def read_csv(path):
    with open(path) as f:
        rd = csv.reader(f)
        head = next(rd, None)
        if head is None:
            raise Error("bench csv: empty input")
        if head[:16] != HEADER:
            raise Error("bench csv: unrecognized header/schema: '%s'" % ",".join(head))
        rows = []
        for line in rd:
            if not line:
                continue
            r = dict(zip(head, line))
            rows.append(dict(bits=int(r["bits"]), u=int(r["u"]), v=int(r["v"]),
                             eff_gflops=float(r["eff_gflops"]), status=r["status"]))
        return rows


def crossover_table(rows):
    """bench.cpp:93-136: per-bitsize winner merged into segments."""
    best, seen_bits, seen_var = {}, set(), set()
    for r in rows:
        seen_bits.add(r["bits"])
        if r["status"] != "ok":
            continue
        seen_var.add((r["u"], r["v"]))
        w = best.get(r["bits"])
        if w is None:
            best[r["bits"]] = r
            continue
        uv, wuv = r["u"] * r["v"], w["u"] * w["v"]
        if r["eff_gflops"] > w["eff_gflops"] or (
                r["eff_gflops"] == w["eff_gflops"] and
                (uv < wuv or (uv == wuv and (r["u"] + r["v"] < w["u"] + w["v"] or
                                            (r["u"] + r["v"] == w["u"] + w["v"] and r["u"] < w["u"]))))):
            best[r["bits"]] = r
    if len(seen_var) < 2:
        raise Error("crossover: need measurements for at least two variants")
    if not seen_bits:
        raise Error("crossover: no rows")
    lo, hi = min(seen_bits), max(seen_bits)
    missing = [b for b in range(lo, hi + 1) if b not in seen_bits]
    if missing:
        raise Error("crossover: sweep has gaps at bitsizes " + ", ".join(map(str, missing)))
    out = []
    for b in range(lo, hi + 1):
        w = best.get(b)
        if w is None:
            continue
        var = (w["u"], w["v"])
        if out and out[-1][0] == var and out[-1][2] == b - 1:
            out[-1][2] = b
        else:
            out.append([var, b, b])
    return out


# ------------------------------------------------------------------- check
CHECK_DIMS = [(17, 33, 9), (64, 64, 64), (128, 300, 32)]
CHECK_BITS = [5, 20, 26, 30, 35, 39, 42, 48, 52]
ORACLE_CAP = 512


def verify_product(A, B, C, p: int, trials: int, samples: int, seed: int):
    """None if C == A B mod p passes `trials` exact Freivalds trials and the
    sampled entries, else a note naming the failure.  Exact Python-integer
    arithmetic; C itself is never recomputed."""
    m, k = A.shape
    n = B.shape[1]
    if m == 0 or n == 0:
        return None
    rng = np.random.default_rng(seed)
    Ai = A.astype(np.int64)
    Bi = B.astype(np.int64)
    Ci = C.astype(np.int64)
    if (Ci < 0).any() or (Ci >= p).any():
        i, j = np.argwhere((Ci < 0) | (Ci >= p))[0]
        return "entry (%d,%d) = %d outside [0, p)" % (i, j, Ci[i, j])
    for (i, j) in zip(rng.integers(0, m, samples), rng.integers(0, n, samples)):
        want = sum(int(Ai[i, t]) * int(Bi[t, j]) for t in range(k)) % p
        if int(Ci[i, j]) != want:
            return "mismatch at (%d,%d): got %d, want %d" % (i, j, int(Ci[i, j]), want)
    Ao, Bo, Co = Ai.astype(object), Bi.astype(object), Ci.astype(object)
    for t in range(trials):
        sv = np.array([int(x) for x in rng.integers(0, p, n, dtype=np.int64)], dtype=object)
        lhs = Co.dot(sv) % p
        rhs = Ao.dot(Bo.dot(sv) % p) % p
        if not (lhs == rhs).all():
            return "Freivalds trial %d failed (row %d)" % (t, int(np.argmax(lhs != rhs)))
    return None


def run_check(args):
    """driver.cpp:37-140: every variant x bitsize x shape x seed against an
    independent check; the planned lambda unless --lambda overrides it."""
    dims = [parse_dims(d) for d in args.dims] if args.dims else CHECK_DIMS
    for d in dims:
        if max(d) > ORACLE_CAP:
            raise Error("check: dims exceed the oracle cap of %d" % ORACLE_CAP)
    variants = parse_variants(args.variant) or [(v.u, v.v) for v in kVariants]
    product = {"plain": mw_product, "concat": mw_product_concat, "workspace": mw_product_workspace}[args.op]
    flags = KERNELS[args.kernel] | (CHECK_EXACTNESS if args.checked else 0)
    passed = failed = skipped = 0
    lines = []
    for (m, k, n) in dims:
        for bits in args.bits:
            for s in range(args.seeds):
                seed = args.seed + s
                p = prev_prime(1 << bits) if 2 <= bits <= 52 else 0
                problem = ""
                if bits > 52:
                    problem = "modulus unrepresentable at t=53"
                elif p < 5 or p.bit_length() != bits:
                    problem = "no usable prime of bitsize %d" % bits
                A = B = None
                for (u, v) in variants:
                    label = "(%d,%d) bits=%d dims=%dx%dx%d seed=%d" % (u, v, bits, m, k, n, seed)
                    status, note = "SKIP", problem
                    if not problem and bits > variant_bit_limit(u, v):
                        note = "skipped (over variant bit limit %d)" % variant_bit_limit(u, v)
                    elif not problem:
                        if A is None:
                            A = random_mat(m, k, p, matrix_seed(seed, bits, m, k, n, 0xA))
                            B = random_mat(k, n, p, matrix_seed(seed, bits, m, k, n, 0xB))
                        lam = args.lambda_ if args.lambda_ else min(mw_block_size(u, v, p), max(k, 1))
                        try:
                            C = product(A, B, u, v, lam, FpContext.make(p), flags=flags)
                            bad = verify_product(A, B, C, p, args.trials, 4, seed * 1000003 + bits)
                            status, note = ("FAIL", bad) if bad else ("PASS", "")
                            if bad and args.dump_dir:
                                import os
                                os.makedirs(args.dump_dir, exist_ok=True)
                                np.save(os.path.join(args.dump_dir, "fail_A.npy"), A)
                                np.save(os.path.join(args.dump_dir, "fail_B.npy"), B)
                        except InfeasibleError as e:
                            status, note = ("FAIL" if args.lambda_ else "SKIP"), str(e)
                        except Error as e:  # e.g. the CHECK_EXACTNESS contract
                            status, note = "FAIL", str(e)
                    passed += status == "PASS"
                    failed += status == "FAIL"
                    skipped += status == "SKIP"
                    if not args.quiet or status == "FAIL":
                        lines.append("%s  %s: %s" % (status, label, note))
    lines.append("check: %d passed, %d failed, %d skipped" % (passed, failed, skipped))
    return failed, lines


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="fpmm-b200", description="exact modular matrix multiplication on B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="measure effective Gflops/s, emit CSV")
    b.add_argument("--scenario", default="square", choices=["square", "unbalanced"])
    b.add_argument("--dims")
    b.add_argument("--scale", type=float, default=1.0)
    b.add_argument("--bits", type=int, nargs="+", default=list(range(20, 53)))
    b.add_argument("--variant", nargs="+", default=["auto"])
    b.add_argument("--lambda", dest="lambda_", default="auto")
    b.add_argument("--kernel", default="b200", choices=sorted(KERNELS))
    b.add_argument("--runs", type=int, default=10)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--out")
    b.add_argument("--extended", action="store_true")
    b.add_argument("--device-resident", action="store_true",
                   help="square scenario with inputs already on the GPU, timed by CUDA events (no PCIe)")
    ck = sub.add_parser("check", help="oracle-equivalence suite (PASS/FAIL/SKIP per case)")
    ck.add_argument("--bits", type=int, nargs="+", default=CHECK_BITS)
    ck.add_argument("--dims", nargs="+")
    ck.add_argument("--variant", nargs="+", default=["auto"])
    ck.add_argument("--op", default="plain", choices=["plain", "concat", "workspace"])
    ck.add_argument("--seed", type=int, default=1)
    ck.add_argument("--seeds", type=int, default=3)
    ck.add_argument("--kernel", default="b200", choices=sorted(KERNELS))
    ck.add_argument("--lambda", dest="lambda_", type=int, default=0)
    ck.add_argument("--checked", action="store_true")
    ck.add_argument("--trials", type=int, default=2)
    ck.add_argument("--dump-dir")
    ck.add_argument("--quiet", action="store_true")
    c = sub.add_parser("crossover", help="best-variant bitsize intervals from a bench CSV")
    c.add_argument("csv")
    c.add_argument("--out")
    pl = sub.add_parser("plan", help="variant/block-size plan for a bitsize and shape")
    pl.add_argument("--bits", type=int, required=True)
    pl.add_argument("--dims", default="1024,1024,1024")
    pl.add_argument("--min-lambda", type=int, default=1)
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 2 if e.code else 0
    try:
        if args.cmd == "bench":
            rows = run_bench(args)
            if args.out:
                with open(args.out, "w") as f:
                    write_csv(rows, f, args.extended)
            else:
                write_csv(rows, sys.stdout, args.extended)
        elif args.cmd == "check":
            failed, lines = run_check(args)
            print("\n".join(lines))
            return 1 if failed else 0
        elif args.cmd == "crossover":
            table = crossover_table(read_csv(args.csv))
            buf = io.StringIO()
            buf.write("u,v,best_bits_lo,best_bits_hi\n")
            for (u, v), lo, hi in table:
                buf.write("%d,%d,%d,%d\n" % (u, v, lo, hi))
            if args.out:
                open(args.out, "w").write(buf.getvalue())
            else:
                sys.stdout.write(buf.getvalue())
        else:
            from . import select_variant
            m, k, n = parse_dims(args.dims)
            p = select_variant(args.bits, m, k, n, min_lambda=args.min_lambda)
            print("bits=%d dims=%d,%d,%d variant=(%d,%d) lambda=%d concat=%s products=%d reductions=%d "
                  "storage=%d" % (args.bits, m, k, n, p.u, p.v, p.lambda_, p.concat, p.predicted_products,
                                  p.predicted_reductions, p.storage_entries))
    except Error as e:
        print("error: %s" % e, file=sys.stderr)
        return 1
    return 0


if __name__ == "__main__":
    sys.exit(main())
