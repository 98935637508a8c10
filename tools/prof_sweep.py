"""Run the C4 sweep on a few scenarios (for ncu / launch lists)."""
import ctypes as C
import sys
import pathlib

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np  # noqa: E402
from cases import c4_spec  # noqa: E402
from paper_2602_22718_b200 import _abi  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402
from paper_2602_22718_b200.rollsim import default_profile  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 148
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = context(0)
prof = default_profile()
ps, keep = prof.struct()
spec = c4_spec(S, count=65536)
Cn = 256
bufs = [np.zeros(S * Cn), np.zeros(S * Cn), np.zeros(S * Cn, np.int64), np.zeros(S, np.int32),
        np.zeros(Cn, np.int32), np.zeros(Cn), np.zeros(Cn)]
ptrs = [b.ctypes.data for b in bufs]
if "noidle" in sys.argv[3:]:
    ptrs[2] = None  # no idle_slot_ticks output
out = _abi.RsSweepOut(*ptrs)
import time
ctx.enable_kernel_timing(True)
for r in range(reps):
    t0 = time.perf_counter()
    ctx.reset_kernel_timing()
    check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, 1, 256, 0.7, 2, C.byref(out), 0))
    print(f"rep {r} wall {1e3 * (time.perf_counter() - t0):.1f} ms")
    for k in ("gen_scenarios", "fast_build", "fast_tables", "group_table", "group_eval", "finish", "candidate_reduce", "select", "aggregate"):
        ms, n = ctx.kernel_time(k)
        print(f"rep {r} {k}: {ms:.3f} ms over {n} launches")
print("n_star[:8]", bufs[3][:8])
