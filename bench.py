#!/usr/bin/env python
"""Benchmark: effective modular GFLOP/s (2mnk / t) of C = A B mod p on B200.

Default workload (BASELINE.json configs[1]): m = n = k = 8192, one product per
prime bitsize 20..52 (p = prev_prime(2^b)), (u, v, lambda) from the paper's
selection rule (plan_for_modulus).  One step = the whole sweep (33 products).
Inputs are synthetic uniform residues generated on the device and resident in
HBM (each 512 MiB operand is larger than the 126 MB L2, so no flush is needed).

  python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference]
                  [--workload sweep8192|c1|c3|c4|c5] [--bits 20-52]

N > 1 runs under torchrun (one process per GPU): A / C row blocks per rank,
B words broadcast over NCCL from rank 0, C gathered on rank 0, all inside the
timed region; the step time is the max over ranks.

`--impl reference` times the reference's own CPU implementation (the
unmodified /root/reference/proj sources compiled into oracle/_ref) on a
bounded sample of the same sweep, on all host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL writes its banner / debug log to stdout; keep stdout to the one JSON
# line the driver parses
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")


class _StdoutToStderr:
    """fd-level redirect of stdout to stderr (NCCL prints its version banner
    with printf at communicator creation)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)
        return False

WORKLOADS = {
    # name: (m, k, n, bits list or None for --bits)
    "sweep8192": (8192, 8192, 8192, None),
    "c1": (1024, 1024, 1024, [50]),
    "c3": (32768, 32768, 32768, [52]),
    "c4": (4096, 262144, 4096, [48]),
    "c5": (65536, 256, 65536, [40]),
}


def parse_bits(s: str):
    out = []
    for part in s.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += list(range(int(a), int(b) + 1))
        elif part:
            out.append(int(part))
    return out


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled during the
    timed region: NVML every 20 ms (nvidia-ml-py), else nvidia-smi every 0.2 s.
    Samples are [sm_mhz, max_mhz, power_w, hw_slowdown, hw_thermal, sw_thermal,
    sw_power_cap]."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        while not self._stop.is_set():
            try:
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)), float(mx),
                                     nv.nvmlDeviceGetPowerUsage(h) / 1000.0] +
                                    [bool(r & b) for b in bits])
            except Exception:
                pass
            self._stop.wait(0.02)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.source = "nvml"
            try:
                return self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    f = [x.strip() for x in out.split(",")]
                    num = lambda x: float(x) if x.replace(".", "").isdigit() else None  # noqa: E731
                    self.samples.append([num(f[0]), num(f[1]), num(f[2])] + [x.lower() == "active" for x in f[3:7]])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = sorted(s[0] for s in self.samples if s[0] is not None)
        mx = max((s[1] for s in self.samples if s[1] is not None), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i]})
        pw = [s[2] for s in self.samples if s[2] is not None]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.samples), "source": self.source, "power_w_max": max(pw) if pw else None}


# --------------------------------------------------------------- reference
# The reference CPU path at 8192^3: the bitsizes whose block
# size lambda >= 255 finish in seconds to a minute on the host; the
# lambda-collapsed ones (lambda <= 31: 24-26, 32-39, 47-52) take hours at
# 8192^3 (the serial per-panel mod-p reduction) and are not
# run.  Excluding them overstates the reference's sweep rate, so the
# driver's GPU/CPU ratio is a lower bound.
REF_BITS_8192 = [20, 21, 22, 27, 28, 29, 30, 40, 41, 42, 43, 44, 45]
REF_WARMUP_DIM = 1024  # warm-up steps: one product at 1024^3 (page-in, BLAS threads)


def reference_product(bits, m, k, n, threads, want_c=False):
    """One product of the reference's run_bench square timed region
    (driver.cpp:222-243: lambda, decompose(B), decompose(A), mw_product_words)
    on the reference's own seeded inputs; returns (2mnk, seconds, C or None)."""
    import ctypes as C

    import numpy as np

    import oracle as O
    R = O.ref()
    if R is None:
        raise RuntimeError("oracle/_ref/libfpmm_ref.so missing")
    R.ref_set_threads(threads)
    p, A, B = O.seeded_inputs(m, k, n, bits)
    pl = O.plan_for_modulus(p, m, k, n)
    Cm = np.empty((m, n))
    t = C.c_double()
    st = R.ref_bench_square(O._ptr(A), O._ptr(B), m, k, n, p, pl.u, pl.v, 1, 1, O._ptr(Cm), C.byref(t))
    if st:
        raise RuntimeError(R.ref_last_error().decode())
    return 2.0 * m * k * n, t.value, ((p, A, B, Cm) if want_c else None)


def run_reference(args, bits_list):
    """--impl reference: each timed step is one 8192^3 reference product,
    cycling through REF_BITS_8192 (the feasible part of the sweep)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    m, k, n, _ = WORKLOADS[args.workload]
    bl = [b for b in REF_BITS_8192 if b in bits_list] if args.workload == "sweep8192" else bits_list
    if not bl:
        bl = bits_list
    dim_note = "%dx%dx%d" % (m, k, n)
    if args.workload != "sweep8192" and m * k * n > 8192 ** 3:
        # C3 / C4 / C5 take hours on the host: a 1024^3 product at the config's bitsize, labelled
        m = k = n = 1024
        dim_note = "1024^3 (the configured shape takes hours on the host)"
    for _ in range(args.warmup):
        reference_product(bl[0], REF_WARMUP_DIM, REF_WARMUP_DIM, REF_WARMUP_DIM, threads)
    F = S = 0.0
    per = {}
    for i in range(args.steps):
        b = bl[i % len(bl)]
        f, s, _ = reference_product(b, m, k, n, threads)
        F += f
        S += s
        per[str(b)] = round(f / s / 1e9, 3)
    v = F / S / 1e9
    sample = ("%d steps, one %s reference product each, bits %s in turn (lambda >= 255 only; the "
              "lambda-collapsed bitsizes take hours at this size); run_bench square timed region "
              "(driver.cpp:222-243), OpenBLAS dgemm on %d threads; warm-up: %d products at %d^3"
              % (args.steps, dim_note, ",".join(str(b) for b in bl), threads, args.warmup, REF_WARMUP_DIM))
    line = {
        "impl": "reference", "metric": "effective modular GFLOP/s (2mnk/s) over the prime-bitsize sweep",
        "value": round(v, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(S / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64 (reference: FP64 dgemm + FP64 reductions)",
        "data": "synthetic (reference random_mat + matrix_seed)",
        "config": {"workload": args.workload, "m": m, "k": k, "n": n, "bits": bl,
                   "rule": "plan_for_modulus (b=2 scan fix)"},
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": sample, "per_bits": per},
        "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- B200
CPU_BASELINE_BITS = [20, 27, 40]  # one 8192^3 reference product per (u,v) class (1,1), (1,2), (2,2)
LINE_MAX = 3000  # the driver keeps a bounded tail of stdout: the JSON line stays well under it


def _detail_path():
    p = os.environ.get("FPMM_BENCH_DETAIL")
    if p:
        return p
    d = os.path.join(ROOT, "gpurun_out")
    return os.path.join(d if os.path.isdir(d) else ROOT, "bench_detail.json")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="sweep8192", choices=sorted(WORKLOADS))
    ap.add_argument("--bits", default="20-52")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the one-process-per-GPU NCCL path even at world size 1 (testing)")
    ap.add_argument("--streams", type=int, default=1,
                    help="streams the sweep's independent products alternate between (N=1); measured: 2-3 "
                         "streams overlap packing/CRT with the tensor kernel but run 3%% slower under the "
                         "1 kW power cap (SM clock 1.49 -> 1.30 GHz)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-engines", action="store_true", help="skip the per-engine recorded passes")
    ap.add_argument("--engine", default="auto", choices=["auto", "i8", "rns", "dmma"],
                    help="engine timed for `value`/`e2e` (auto = the library default; all are recorded per "
                         "bitsize)")
    args = ap.parse_args()
    m, k, n, wl_bits = WORKLOADS[args.workload]
    bits_list = wl_bits if wl_bits is not None else parse_bits(args.bits)
    if args.impl == "reference":
        return run_reference(args, bits_list)
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps

    import numpy as np
    import torch

    import paper_2601_07508_b200 as F
    from paper_2601_07508_b200 import dist as D

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and "RANK" in os.environ:
        print("warning: WORLD_SIZE %d != --gpus %d" % (world, args.gpus), file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    part = None
    # the one-process-per-GPU path (NCCL broadcast of B, gather of C); --force-dist
    # runs it at world size 1 too (under torchrun --nproc-per-node 1), as a test
    dist = world > 1 or args.force_dist
    if dist:
        import torch.distributed as td
        with _StdoutToStderr():
            td.init_process_group("nccl", device_id=dev)
            part = D.init_from_torch(local)

    # problems of the step: (bits, p, u, v, lambda, lambda_k)
    probs = []
    for b in bits_list:
        p = F.prev_prime(1 << b)
        pl = F.plan_for_modulus(p, m, k, n)
        probs.append((b, p, pl.u, pl.v, pl.lambda_, F.kernel_block(p, pl.u, pl.v)))

    # resident inputs and outputs, one set per bitsize: each rank holds its A
    # row block and C row block, B lives on rank 0, the gathered C on rank 0.
    # Every product of a step writes its own C, so the outputs of the last
    # timed step are all verified afterwards.
    A, B, Cr, Cf, rows = {}, {}, {}, {}, {}
    for (b, p, u, v, lam, _) in probs:
        r0, rn = part.rows_for(m, u, v) if part else (0, m)
        rows[b] = (r0, rn)
        A[b] = torch.empty((max(rn, 1), k), dtype=torch.float64, device=dev)
        F.random_residues_device(A[b][:rn] if rn else A[b][:0], p, F.matrix_seed(1, b, m, k, n, 0xA), row0=r0)
        if rank == 0:
            B[b] = torch.empty((k, n), dtype=torch.float64, device=dev)
            F.random_residues_device(B[b], p, F.matrix_seed(1, b, m, k, n, 0xB))
        if dist:
            Cr[b] = torch.empty((max(rn, 1), n), dtype=torch.float64, device=dev)
            Cf[b] = torch.empty((m, n), dtype=torch.float64, device=dev) if rank == 0 else None
        else:
            Cf[b] = torch.empty((m, n), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    # measured tensor-pipe peaks of this GPU (MEASURED_PEAKS.json has neither)
    # int8: burst (short) and sustained (1.4 s of random-operand MMAs: the power
    # cap, not the tensor pipe, bounds a long int8 step on this 1 kW part)
    peaks = {"dmma": F.fp64_peak(local), "i8_burst": F.i8_peak(local, 200000),
             "i8": F.i8_peak(local, 20000000)}
    eng_flags = {"dmma": F.ENGINE_DMMA, "i8": F.ENGINE_I8, "rns": F.ENGINE_RNS, "auto": 0}
    # one non-default stream carries every product and the timing events
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    nstreams = max(1, args.streams) if not dist else 1
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nstreams - 1)]
    launches = [0]
    per_launch = {}

    def step(engine, record=None):
        fl = eng_flags[engine] | (0 if record is not None else F.ASYNC)
        for idx, (b, p, u, v, lam, _) in enumerate(probs):
            tm = F.Timing()
            if not dist:
                sidx = idx % nstreams if record is None else 0
                F.mw_product_device(A[b], B[b], Cf[b], p, u, v, lam, stream=streams[sidx], flags=fl,
                                    timing=tm if record is not None else None)
            else:
                r0, rn = rows[b]
                D.mw_product_device(A[b][:rn], B.get(b), Cr[b][:rn], p, u, v, lam, m, root=0,
                                    C_full=Cf[b], stream=stream, flags=fl,
                                    timing=tm if record is not None else None)
            launches[0] += per_launch.get(b, 0)
            if record is not None:
                record[b] = (tm.gemm_ms, tm.engine, tm.words, tm.launches, tm.recon_ms, tm.pack_ms, tm.lambda_k)

    def barrier():
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    vtmp = {}

    def verify_all(tag):
        """Exact device check of every product's C (on rank 0): range,
        2 Freivalds trials mod p, 64 sampled exact entries.  Outside timing."""
        out = {}
        if rank != 0:
            return out
        for (b, p, u, v, lam, _) in probs:
            if dist and world > 1:
                # the full A for the check (each rank holds a row block)
                Af = vtmp.get("A")
                if Af is None or tuple(Af.shape) != (m, k):
                    Af = vtmp["A"] = torch.empty((m, k), dtype=torch.float64, device=dev)
                F.random_residues_device(Af, p, F.matrix_seed(1, b, m, k, n, 0xA), row0=0, stream=stream)
            else:
                Af = A[b][:m]
            r = F.verify_device(Af, B[b], Cf[b], p, seed=1000 + b, trials=2, samples=64, stream=stream)
            out[str(b)] = r["ok"]
            if not r["ok"]:
                print("VERIFY FAILED (%s) bits=%d: %s" % (tag, b, r), file=sys.stderr)
        return out

    # first warm-up step recorded: each product's kernel-launch count (tm.launches)
    rec0 = {}
    step(args.engine, record=rec0)
    per_launch.update({b: r[3] for b, r in rec0.items()})
    for _ in range(args.warmup - 1):
        step(args.engine)
    barrier()
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        e0.record(stream)
        for s_ in streams[1:]:
            s_.wait_event(e0)
        for _ in range(args.steps):
            step(args.engine)
        for s_ in streams[1:]:
            ev_ = torch.cuda.Event()
            ev_.record(s_)
            stream.wait_event(ev_)
        e1.record(stream)
        barrier()
    elapsed_ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([elapsed_ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    timed_launches = launches[0]
    # the outputs of the last timed step, every product
    verified = verify_all("timed")
    barrier()

    flops_step = sum(2.0 * m * k * n for _ in probs)
    ms_per_step = elapsed_ms / args.steps
    value = flops_step / (ms_per_step * 1e-3) / 1e9

    # one recorded pass per engine (library CUDA events around the GEMM kernel
    # on the launching stream): per-bitsize table and each kernel's roofline
    traffic_db = {}
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic_db = json.load(open(prof))
        except Exception:
            traffic_db = {}
    engines = {}
    kernel_desc = {
        F.ENGINE_DMMA: "mwgemm_kernel: DMMA.8x8x4 FP64 tensor pipe; work = 2uv*mnk FP64 flops",
        F.ENGINE_I8: "mwi8_kernel: tcgen05.mma.kind::i8 (UTCIMMA), TMEM int32; work = 2*D^2*mnk int8 tensor "
                     "ops (D base-256 digits)",
        F.ENGINE_RNS: "rns_kernel: tcgen05.mma.cta_group::2.kind::i8 (UTCIMMA.2CTA) M256 N256, TMEM int32, "
                      "CRT in the last modulus pass's epilogue; work = 2*n_mod*mnk int8 tensor ops",
    }
    eng_verified = {}
    eng_list = [args.engine] if args.no_engines else ["auto", "i8", "rns", "dmma"]
    for eng in eng_list:
        rec = {}
        if eng != args.engine:
            step(eng)  # untimed: first launches of this engine's kernels (lazy module loading)
        step(eng, record=rec)
        torch.cuda.synchronize()
        eng_verified[eng] = verify_all(eng)
        per_bits = {}
        work = gemm_total = 0.0
        ran = set()
        for (b, p, u, v, lam, lk) in probs:
            g, e_ran, words, _, recon, packt, lk_run = rec[b]
            ran.add(e_ran)
            rn = rows[b][1]
            if e_ran == F.ENGINE_DMMA:
                w = 2.0 * u * v * rn * k * n           # uv-scaled FP64 work (the rule's words)
                # FP64-pipe ceiling: the engine's words (`words` = u'v') reduce every lambda_k' terms
                # with 3 FP64-pipe ops, so at most lambda_k'/(lambda_k'+3) of the pipe does DMMA
                ceil_uv = (u * v / words) * lk_run / (lk_run + 3.0) if words and lk_run else None
                extra = {"lambda_k": lk_run, "engine_uv": words,
                         "ceiling": round(ceil_uv, 4) if ceil_uv else None}
            elif e_ran == F.ENGINE_I8:
                w = 2.0 * words * words * rn * k * n   # D^2 int8 digit products
                extra = {"engine": "i8", "digits": words}
            else:
                w = 2.0 * words * rn * k * n           # one int8 GEMM per byte modulus
                extra = {"engine": "rns", "moduli": words}
            work += w
            gemm_total += g
            pk = "dmma" if e_ran == F.ENGINE_DMMA else "i8"
            per_bits[str(b)] = dict({"u": u, "v": v, "lambda": lam, "gemm_ms": round(g, 3),
                                     "pack_ms": round(packt, 3), "recon_ms": round(recon, 3),
                                     "eff_gflops": round(2.0 * rn * k * n / (g * 1e-3) / 1e9, 1),
                                     "tensor_frac": round(w / (g * 1e-3) / 1e12 / peaks[pk], 4)}, **extra)
        achieved = work / (gemm_total * 1e-3) / 1e12
        pk = "dmma" if eng == "dmma" else "i8"
        tr = traffic_db.get(eng, {})
        engines[eng] = {
            "eff_gflops": round(flops_step / (gemm_total * 1e-3) / 1e9, 1),
            "roofline": {"bound": "tensor", "achieved": round(achieved, 3), "peak": round(peaks[pk], 3),
                         "unit": "TFLOP/s", "frac": round(achieved / peaks[pk], 4),
                         "traffic": tr.get("dram_bytes_per_launch"),
                         "traffic_source": tr.get("source"),
                         "kernel": " + ".join(kernel_desc[e] for e in sorted(ran)),
                         "peak_source": ("measured DMMA-only loop on this GPU (MEASURED_PEAKS.json has no FP64 "
                                         "entry); vendor FP64 tensor 37.2 TF @1965 MHz" if pk == "dmma" else
                                         "measured SUSTAINED tcgen05 kind::i8 rate on this GPU (1.4 s of "
                                         "M128 N256 K32 MMAs under the 1 kW cap; MEASURED_PEAKS.json has no "
                                         "int8 entry); burst %.0f TOP/s" % peaks["i8_burst"])},
            "sweep": per_bits}
        if pk == "i8":
            engines[eng]["roofline"]["frac_of_burst_peak"] = round(achieved / peaks["i8_burst"], 4)
    roof = dict(engines[args.engine]["roofline"])
    # HBM rooflines of the RNS engine's memory-side kernels over the sweep
    # (north star: achieved HBM GB/s of the decomposition): the packs read 8 B
    # and write n_mod B per operand element.  Times are the library's CUDA
    # events around them.
    hbm_peak = None
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    memside = {}
    if "rns" in engines:
        rs = engines["rns"]["sweep"]
        pk_b = pk_t = cr_b = cr_t = 0.0
        for (b, p, u, v, lam, lk) in probs:
            e = rs[str(b)]
            nm = e.get("moduli", 0)
            rn = rows[b][1]
            pk_b += (8.0 + nm) * (rn * k + k * n)
            pk_t += e["pack_ms"]
            cr_b += (nm + 8.0) * rn * n
            cr_t += e["recon_ms"]
        for key, by, t, kern in (("decomposition", pk_b, pk_t, "pack_a_rns + pack_b_rns_direct"),
                                 ("reconstruction", cr_b, cr_t, "rns_crt_kernel (split-K products only)")):
            if t > 0:
                gbs = by / (t * 1e-3) / 1e9
                memside[key] = {"kernel": kern, "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                                "unit": "GB/s", "frac": round(gbs / hbm_peak, 4) if hbm_peak else None,
                                "ms_per_step": round(t, 3)}
    # FP64 path (north star): uv-adjusted fraction of the measured DMMA peak,
    # and the bitsizes below the 70% target with their FP64-pipe ceiling
    fp64 = None
    if "dmma" in engines:
        sw = engines["dmma"]["sweep"]
        fp64 = {"uv_frac": engines["dmma"]["roofline"]["frac"], "peak_tflops": round(peaks["dmma"], 2),
                "below_70pct": {b: [e["tensor_frac"], e.get("ceiling")] for b, e in sw.items()
                                if e["tensor_frac"] < 0.70},
                "note": "[uv-adjusted frac, FP64-pipe ceiling uv/u'v' * lk/(lk+3)] per bitsize"}
    # end to end through the public host-buffer API (pinned memory), one step
    e2e = None
    e2e_trace = None
    if not args.no_e2e:
        e2e, e2e_trace = run_e2e(F, D, torch, np, probs, A, B, Cf, rows, m, k, n, dist, rank, part,
                                 eng_flags[args.engine])

    cpu = None
    cpu_detail = None
    if rank == 0 and world == 1 and not args.no_cpu and args.workload == "sweep8192":
        try:
            cpu, cpu_detail = run_cpu_baseline(F, torch, np, m, k, n, [b for b in CPU_BASELINE_BITS if b in bits_list],
                                               eng_flags[args.engine], stream)
        except Exception as ex:  # reported, never silently substituted
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                   "sample": "unavailable: %s" % ex}

    if rank == 0:
        nver = sum(1 for x in verified.values() if x)
        all_ok = nver == len(probs) and all(all(d.values()) for d in eng_verified.values())
        clocks = clk.summary()
        detail = {"value": value, "ms_per_step": ms_per_step, "engine": args.engine, "engines": engines,
                  "memory_side": memside, "fp64": fp64, "e2e": e2e, "e2e_trace": e2e_trace, "cpu_baseline": cpu,
                  "cpu_detail": cpu_detail, "verified_timed": verified, "verified_engines": eng_verified,
                  "clocks": clocks, "peaks": peaks}
        dpath = _detail_path()
        try:
            with open(dpath, "w") as f:
                json.dump(detail, f, indent=1)
        except Exception as ex:
            print("could not write %s: %s" % (dpath, ex), file=sys.stderr)
        roof.pop("kernel", None)
        roof["kernel"] = "rns_kernel" if "rns" in json.dumps(engines[args.engine]["sweep"]) else "auto"
        line = {
            "metric": "effective modular GFLOP/s (2mnk/s) over the prime-bitsize sweep",
            "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 in/out (exact residues); int8 tcgen05 residue GEMMs (u8 x u8 -> s32)",
            "data": "synthetic uniform residues (device splitmix64), resident in HBM",
            "config": {"workload": args.workload, "m": m, "k": k, "n": n,
                       "bits": [bits_list[0], bits_list[-1]], "products_per_step": len(probs),
                       "parallelism": "row-sharded x%d" % world, "l2": "inputs 512 MiB/operand > L2; no flush"},
            "verified": {"ok": all_ok, "timed_products": nver, "of": len(probs),
                         "method": "device: C in [0,p), 2 Freivalds trials mod p, 64 exact entries"},
            "roofline": roof,
            "fp64_uv_frac": fp64["uv_frac"] if fp64 else None,
            "memory_side": {k_: {"achieved": v_["achieved"], "frac": v_["frac"]} for k_, v_ in memside.items()},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": timed_launches,
            "clocks": {k_: clocks.get(k_) for k_ in ("sm_mhz", "sm_max_mhz", "reasons")},
            "detail": os.path.relpath(dpath, ROOT),
        }
        txt = json.dumps(line)
        for drop in ("memory_side", "fp64_uv_frac", "detail"):  # keep the line short for the driver
            if len(txt) <= LINE_MAX:
                break
            line.pop(drop, None)
            txt = json.dumps(line)
        if len(txt) > LINE_MAX and cpu:
            line["cpu_baseline"] = {k_: cpu.get(k_) for k_ in ("value", "unit", "cores", "kind")}
            txt = json.dumps(line)
        print(txt, flush=True)
    if dist:
        D.finalize()
        torch.distributed.destroy_process_group()


def run_cpu_baseline(F, torch, np, m, k, n, bits_list, flags, stream):
    """cpu_baseline leg (rank 0, N=1): one 8192^3 reference product per
    listed bitsize on the reference's own seeded inputs, timed like run_bench
    (driver.cpp:222-243); the same inputs then go through the GPU product,
    whose C must equal the reference's bit for bit, and are timed on the
    device for a same-size GPU/CPU ratio."""
    threads = os.cpu_count() or 1
    F_ = S = 0.0
    per = {}
    for b in bits_list:
        f, s, (p, Ah, Bh, Cref) = reference_product(b, m, k, n, threads, want_c=True)
        F_ += f
        S += s
        pl = F.plan_for_modulus(p, m, k, n)
        dA = torch.from_numpy(Ah).to("cuda")
        dB = torch.from_numpy(Bh).to("cuda")
        dC = torch.empty((m, n), dtype=torch.float64, device="cuda")
        F.mw_product_device(dA, dB, dC, p, pl.u, pl.v, pl.lambda_, stream=stream, flags=flags)
        same = bool(np.array_equal(dC.cpu().numpy(), Cref))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        F.mw_product_device(dA, dB, dC, p, pl.u, pl.v, pl.lambda_, stream=stream, flags=flags | F.ASYNC)
        e1.record(stream)
        e1.synchronize()
        g = e0.elapsed_time(e1)
        per[str(b)] = {"cpu_gflops": round(f / s / 1e9, 2), "cpu_s": round(s, 3),
                       "gpu_gflops": round(f / (g * 1e-3) / 1e9, 1), "gpu_over_cpu": round(s * 1e3 / g, 1),
                       "C_equal_to_reference": same}
        del dA, dB, dC
    v = F_ / S / 1e9
    cpu = {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
           "sample": "one 8192^3 product per bitsize %s through the reference's decompose + mw_product_words "
                     "(driver.cpp:222-243 timed region), OpenBLAS dgemm on %d threads, %.1f s; the GPU C "
                     "equals the reference's: %s" % (bits_list, threads, S,
                                                     all(x["C_equal_to_reference"] for x in per.values()))}
    return cpu, per


def run_e2e(F, D, torch, np, probs, A, B, Cf, rows, m, k, n, dist, rank, part, flags):
    """E: the sweep through the host-buffer public API.  Each product's timed
    region covers H2D of its inputs from pinned memory, the product and the
    D2H of C.  Inputs are staged into the pinned buffers outside the timer."""
    pin = lambda shape: torch.empty(shape, dtype=torch.float64, pin_memory=True)  # noqa: E731
    maxrows = max(r[1] for r in rows.values())
    hA = pin((max(maxrows, 1), k))
    hB = pin((k, n)) if rank == 0 else None
    hC = pin((m, n)) if rank == 0 else None
    hA.zero_()
    if hB is not None:
        hB.zero_()
    secs = 0.0
    h2d = d2h = 0
    flops = 0.0
    scratch = {"n": n}
    trace = []
    # untimed warm-up pass over the sweep: the library's staging buffers and
    # workspaces grow to the largest product (the RNS moduli count rises with
    # the bitsize, and a grow is a cudaFree + cudaMalloc that serialises the
    # device), so the timed pass measures the steady state
    for (b, p, u, v, lam, _) in probs:
        r0, rn = rows[b]
        if not dist:
            F.mw_product(hA[:rn].numpy(), hB.numpy(), u, v, lam, F.FpContext.make(p), out=hC.numpy(), flags=flags)
        else:
            D.mw_product_host(hA[:rn], hB, hC, p, u, v, lam, m, root=0, scratch=scratch, flags=flags)
    for (b, p, u, v, lam, _) in probs:
        r0, rn = rows[b]
        hA[:rn].copy_(A[b][:rn])
        if rank == 0:
            hB.copy_(B[b])
        torch.cuda.synchronize()
        if dist:
            torch.distributed.barrier()
        tm = F.Timing()
        t0 = time.perf_counter()
        if not dist:
            F.mw_product(hA.numpy(), hB.numpy(), u, v, lam, F.FpContext.make(p), out=hC.numpy(),
                         flags=flags, timing=tm)
        else:
            D.mw_product_host(hA[:rn], hB, hC, p, u, v, lam, m, root=0, scratch=scratch, flags=flags)
            torch.distributed.barrier()
        dt = time.perf_counter() - t0
        if dist:
            t = torch.tensor([dt], device="cuda")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            dt = float(t.item())
        secs += dt
        trace.append((b, round(dt * 1e3, 2), round(tm.h2d_ms, 2), round(tm.total_ms, 2)))
        flops += 2.0 * m * k * n
        h2d += 8 * (m * k + k * n)
        d2h += 8 * m * n
    Cf_last = Cf.get(probs[-1][0]) if probs else None
    # the host result of the last product equals the device path's output (verified above)
    same = None
    if rank == 0:
        same = bool(torch.equal(hC, Cf_last.cpu())) if Cf_last is not None else None
    return ({"value": round(flops / secs / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
             "d2h_bytes_per_step": d2h, "ms_per_step": round(secs * 1e3, 3), "C_equal_to_device_path": same,
             "api": "mw_product (host pinned)" if not dist else "dist.mw_product_host"}, trace)

if __name__ == "__main__":
    main()
