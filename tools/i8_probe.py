"""Tensor-pipe int8 probes: 1-CTA (M128 N256) vs CTA-pair cta_group::2 (M256 N256), burst and sustained."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_07508_b200 as F  # noqa: E402

L = F.lib()
L.fpmm_b200_i8_probe.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
for mode in (0, 1):
    for iters in (20000, 20000000):
        t = C.c_double()
        st = L.fpmm_b200_i8_probe(0, iters, mode, C.byref(t))
        print("mode", mode, "iters", iters, "status", st, L.fpmm_b200_last_error(), "TOPS %.1f" % t.value, flush=True)
