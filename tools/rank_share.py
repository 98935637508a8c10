"""One rank's share of the C4 sweep at N GPUs (10,000 / N scenarios) timed on
one GPU: the scaling the driver's N-GPU run can reach (max over ranks)."""
import ctypes as C
import pathlib
import sys
import time

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np  # noqa: E402
from cases import c4_spec  # noqa: E402
from paper_2602_22718_b200 import _abi  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402
from paper_2602_22718_b200.rollsim import default_profile  # noqa: E402

ctx = context(0)
ps, keep = default_profile().struct()
for n in (1, 2, 4, 8):
    S = 10000 // n
    spec = c4_spec(S, count=65536)
    Cn = 256
    bufs = [np.zeros(S * Cn), np.zeros(S * Cn), np.zeros(S * Cn, np.int64), np.zeros(S, np.int32),
            np.zeros(Cn, np.int32), np.zeros(Cn), np.zeros(Cn)]
    out = _abi.RsSweepOut(*[b.ctypes.data for b in bufs])
    best = 1e9
    for r in range(3):
        ctx.synchronize()
        t0 = time.perf_counter()
        check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, 1, 256, 0.7, 2, C.byref(out), 0))
        best = min(best, time.perf_counter() - t0)
    print(f"N={n}: {S} scenarios per rank in {best * 1e3:.1f} ms -> {10000 * 256 / best / 1e6:.1f} M evals/s whole job")
