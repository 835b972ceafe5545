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
CPU_SAMPLE_DIM = 512  # reference CPU sample: the same bitsize sweep at 512^3


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
def reference_sweep(bits_list, dim, threads):
    """One pass of the reference's run_bench square timed region (driver.cpp:222-243)
    over bits_list at dim^3; returns (sum 2mnk, sum seconds, per-bit)."""
    import ctypes as C

    import numpy as np

    import oracle as O
    R = O.ref()
    if R is None:
        raise RuntimeError("oracle/_ref/libfpmm_ref.so missing")
    R.ref_set_threads(threads)
    flops = secs = 0.0
    per = {}
    for bits in bits_list:
        p, A, B = O.seeded_inputs(dim, dim, dim, bits)
        pl = O.plan_for_modulus(p, dim, dim, dim)
        Cm = np.empty((dim, dim))
        t = C.c_double()
        st = R.ref_bench_square(O._ptr(A), O._ptr(B), dim, dim, dim, p, pl.u, pl.v, 1, 1, O._ptr(Cm),
                                C.byref(t))
        if st:
            raise RuntimeError(R.ref_last_error().decode())
        flops += 2.0 * dim ** 3
        secs += t.value
        per[bits] = round(2.0 * dim ** 3 / t.value / 1e9, 3)
    return flops, secs, per


def run_reference(args, bits_list):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    sample = "m=n=k=%d, bits %d-%d (%d products), reference mw_product_words + decompose, " \
             "OpenBLAS dgemm, %d threads" % (CPU_SAMPLE_DIM, bits_list[0], bits_list[-1], len(bits_list), threads)
    for _ in range(args.warmup):
        reference_sweep(bits_list, CPU_SAMPLE_DIM, threads)
    F = S = 0.0
    per = None
    for _ in range(args.steps):
        f, s, per = reference_sweep(bits_list, CPU_SAMPLE_DIM, threads)
        F += f
        S += s
    v = F / S / 1e9
    m, k, n, _ = WORKLOADS[args.workload]
    line = {
        "impl": "reference", "metric": "effective modular GFLOP/s (2mnk/s) over the prime-bitsize sweep",
        "value": round(v, 3), "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(S / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference random_mat)",
        "config": {"workload": args.workload, "m": m, "k": k, "n": n, "bits": [bits_list[0], bits_list[-1]],
                   "sample_dim": CPU_SAMPLE_DIM, "rule": "plan_for_modulus (b=2 scan fix)"},
        "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                         "sample": sample, "per_bits": per},
        "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- B200
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

    # problems of the step: (bits, p, u, v, lambda)
    probs = []
    for b in bits_list:
        p = F.prev_prime(1 << b)
        pl = F.plan_for_modulus(p, m, k, n)
        probs.append((b, p, pl.u, pl.v, pl.lambda_, F.kernel_block(p, pl.u, pl.v)))

    # resident inputs: each rank holds its A row block; B lives on rank 0
    A, B, Cr, rows = {}, {}, {}, {}
    for (b, p, u, v, lam, _) in probs:
        r0, rn = part.rows_for(m, u, v) if part else (0, m)
        rows[b] = (r0, rn)
        A[b] = torch.empty((max(rn, 1), k), dtype=torch.float64, device=dev)
        F.random_residues_device(A[b][:rn] if rn else A[b][:0], p, F.matrix_seed(1, b, m, k, n, 0xA), row0=r0)
        if rank == 0:
            B[b] = torch.empty((k, n), dtype=torch.float64, device=dev)
            F.random_residues_device(B[b], p, F.matrix_seed(1, b, m, k, n, 0xB))
    Cbuf = torch.empty((m, n), dtype=torch.float64, device=dev) if rank == 0 else None
    Crow = torch.empty((max(max(r[1] for r in rows.values()), 1), n), dtype=torch.float64, device=dev)
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
    # optionally, independent products alternate between streams (each with its
    # own library workspaces) so one product's packing / CRT runs beside
    # another's tensor-core kernel; one stream under torchrun (NCCL ops in order)
    nstreams = max(1, args.streams) if not dist else 1
    streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(nstreams - 1)]
    Cbufs = [Cbuf] + ([torch.empty_like(Cbuf) for _ in range(nstreams - 1)] if Cbuf is not None else [])
    launches = [0]
    per_launch = {}

    def step(engine, record=None):
        fl = eng_flags[engine] | (0 if record is not None else F.ASYNC)
        for idx, (b, p, u, v, lam, _) in enumerate(probs):
            tm = F.Timing()
            if not dist:
                sidx = idx % nstreams if record is None else 0
                F.mw_product_device(A[b], B[b], Cbufs[sidx], p, u, v, lam, stream=streams[sidx], flags=fl,
                                    timing=tm if record is not None else None)
                launches[0] += per_launch.get(b, 0)
            else:
                r0, rn = rows[b]
                D.mw_product_device(A[b][:rn], B.get(b), Crow[:rn], p, u, v, lam, m, root=0,
                                    C_full=Cbuf, stream=stream, flags=fl,
                                    timing=tm if record is not None else None)
                launches[0] += per_launch.get(b, 0)
            if record is not None:
                record[b] = (tm.gemm_ms, tm.engine, tm.words, tm.launches, tm.recon_ms, tm.pack_ms)

    def barrier():
        if dist:
            torch.distributed.barrier()
        torch.cuda.synchronize()

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
        F.ENGINE_RNS: "rns_kernel: tcgen05.mma.cta_group::2.kind::i8 (UTCIMMA.2CTA) M256 N256, TMEM int32; the "
                      "epilogue parks T_i mod m_i (rns_crt_kernel rebuilds C); work = 2*n_mod*mnk int8 tensor ops "
                      "(n_mod byte moduli)",
    }
    for eng in ("auto", "i8", "rns", "dmma"):
        rec = {}
        if eng != args.engine:
            step(eng)  # untimed: first launches of this engine's kernels (lazy module loading)
        step(eng, record=rec)
        torch.cuda.synchronize()
        per_bits = {}
        work = gemm_total = 0.0
        ran = set()
        for (b, p, u, v, lam, lk) in probs:
            g, e_ran, words, _, recon, packt = rec[b]
            ran.add(e_ran)
            rn = rows[b][1]
            if e_ran == F.ENGINE_DMMA:
                w = 2.0 * u * v * rn * k * n           # uv-scaled FP64 work
                extra = {"lambda_k": lk}
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
                         "kernel": " + ".join(kernel_desc[e] for e in sorted(ran)),
                         "peak_source": ("measured DMMA-only loop on this GPU (MEASURED_PEAKS.json has no FP64 "
                                         "entry); vendor FP64 tensor 37.2 TF @1965 MHz" if pk == "dmma" else
                                         "measured SUSTAINED rate of back-to-back tcgen05 kind::i8 M128 N256 "
                                         "K32 MMAs on random operands, all SMs, 1.4 s under the 1 kW power cap "
                                         "(the kernel is timed inside a long step; MEASURED_PEAKS.json has no "
                                         "int8 entry); burst %.0f TOP/s, vendor dense int8 4.5 POPS"
                                         % peaks["i8_burst"])},
            "sweep": per_bits}
        if pk == "i8":
            engines[eng]["roofline"]["frac_of_burst_peak"] = round(achieved / peaks["i8_burst"], 4)
    roof = dict(engines[args.engine]["roofline"])
    # HBM rooflines of the RNS engine's memory-side kernels over the sweep
    # (north star: achieved HBM GB/s of the decomposition): the packs read 8 B
    # and write n_mod B per operand element; the CRT reads n_mod B and writes
    # 8 B per output element.  Times are the library's CUDA events around them.
    hbm_peak = None
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        pass
    memside = {}
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
    for key, by, t, kern in (("decomposition", pk_b, pk_t, "pack_a_rns + pack_b_rns_direct (A and B residue planes)"),
                             ("reconstruction", cr_b, cr_t, "rns_crt_kernel (parked residues -> C)")):
        if t > 0:
            gbs = by / (t * 1e-3) / 1e9
            memside[key] = {"kernel": kern, "bound": "hbm", "achieved": round(gbs, 1), "peak": hbm_peak,
                            "unit": "GB/s", "frac": round(gbs / hbm_peak, 4) if hbm_peak else None,
                            "bytes_per_step": int(by), "ms_per_step": round(t, 3),
                            "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write)"}
    # end to end through the public host-buffer API (pinned memory), one step
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(F, D, torch, np, probs, A, B, rows, m, k, n, dist, rank, part,
                      eng_flags[args.engine])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = os.cpu_count() or 1
            f, s, per = reference_sweep(bits_list, CPU_SAMPLE_DIM, threads)
            cpu = {"value": round(f / s / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": "reference",
                   "sample": "one pass of the bitsize sweep %d-%d at m=n=k=%d through the reference's "
                             "mw_product_words + decompose (driver.cpp:222-243 timed region), OpenBLAS "
                             "dgemm on %d threads, %.1f s" % (bits_list[0], bits_list[-1], CPU_SAMPLE_DIM,
                                                              threads, s)}
        except Exception as ex:  # reported, never silently substituted
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 0, "kind": "reference",
                   "sample": "unavailable: %s" % ex}

    if rank == 0:
        line = {
            "metric": "effective modular GFLOP/s (2mnk/s) over the prime-bitsize sweep",
            "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic uniform residues (device splitmix64 generator), resident in HBM",
            "config": {"workload": args.workload, "m": m, "k": k, "n": n,
                       "bits": [bits_list[0], bits_list[-1]], "products_per_step": len(probs),
                       "rule": "plan_for_modulus (paper bound, b=2 scan fix)",
                       "parallelism": "row-sharded x%d, NCCL bcast of B (packed words or raw residues, the smaller) + gather C" % world,
                       "l2": "inputs (512 MiB/operand) larger than L2; no flush",
                       "streams": nstreams},
            "engine": args.engine,
            "roofline": roof,
            "fp64_uv_frac": engines["dmma"]["roofline"]["frac"],
            "memory_side": memside,
            "engines": engines,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": timed_launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    if dist:
        D.finalize()
        torch.distributed.destroy_process_group()


def run_e2e(F, D, torch, np, probs, A, B, rows, m, k, n, dist, rank, part, flags):
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
    if os.environ.get("FPMM_BENCH_E2E_TRACE"):
        print("e2e per call (bits, wall ms, library h2d ms, library total ms):", trace, file=sys.stderr)
    return {"value": round(flops / secs / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(secs * 1e3, 3),
            "api": "paper_2601_07508_b200.mw_product (host pinned buffers)" if not dist
            else "paper_2601_07508_b200.dist.mw_product_host"}


if __name__ == "__main__":
    main()
