"""Phase breakdown of fast_build (ns per scenario, thread 0 of each CTA) and
lockstep_eval (SM cycles per warp in phase 1 / phase 2) from the profiling
build: RS_B200_LIB=build/librs_b200_prof.so python tools/phases.py [S]."""
import ctypes as C
import os
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np  # noqa: E402
from cases import c4_spec  # noqa: E402
from paper_2602_22718_b200 import _abi  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402
from paper_2602_22718_b200.rollsim import default_profile  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
ctx = context(0)
lib = ctx.lib
fn = lib.rs_debug_phases
fn.argtypes = [C.POINTER(C.c_ulonglong), C.c_int, C.c_int]
buf = (C.c_ulonglong * 32)()
prof = default_profile()
ps, keep = prof.struct()
spec = c4_spec(S, count=65536)
Cn = 256
bufs = [np.zeros(S * Cn), np.zeros(S * Cn), np.zeros(S * Cn, np.int64), np.zeros(S, np.int32),
        np.zeros(Cn, np.int32), np.zeros(Cn), np.zeros(Cn)]
out = _abi.RsSweepOut(*[b.ctypes.data for b in bufs])
for rep in range(2):
    fn(buf, 32, 1)
    check(lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, 1, 256, 0.7, 2, C.byref(out), 0))
fn(buf, 32, 0)
names = ["gen+hist", "scan+seg", "scatter", "win plan", "win sort+max", "range-max"]
tot = sum(buf[i] for i in range(6))
print(f"fast_build per scenario (us, thread 0): total {tot / S / 1e3:.1f}")
for i, n in enumerate(names):
    print(f"  {n:14s} {buf[i] / S / 1e3:8.2f} us  {100 * buf[i] / max(tot, 1):5.1f}%")
w = S * 8  # warps
p1, p2 = buf[8], buf[9]
print(f"lockstep per warp: phase1 {p1 / w / 1e3:.1f} kcycles, phase2 {p2 / w / 1e3:.1f} kcycles "
      f"({100 * p1 / max(p1 + p2, 1):.1f}% / {100 * p2 / max(p1 + p2, 1):.1f}%)")
