"""Round cost of the lockstep evaluator at c resident CTAs per SM: one
sweep batch of S = 148 * c full-size C4 scenarios per call (one round),
group_eval CUDA-event time (the planner's lockstep_round_cost model)."""
import ctypes as C
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np  # noqa: E402
from cases import c4_spec  # noqa: E402
from paper_2602_22718_b200 import _abi  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402
from paper_2602_22718_b200.rollsim import default_profile  # noqa: E402

ctx = context(0)
ps, keep = default_profile().struct()
base = None
for c in (1, 2, 3, 4):
    S = 148 * c
    spec = c4_spec(S, count=65536)
    out = _abi.RsSweepOut(None, None, None, None, None, None, None)
    bufs = [np.zeros(S * 256), np.zeros(S * 256), np.zeros(S, np.int32)]
    out = _abi.RsSweepOut(bufs[0].ctypes.data, bufs[1].ctypes.data, None, bufs[2].ctypes.data,
                          None, None, None)
    ctx.enable_kernel_timing(True)
    res = []
    for r in range(3):
        ctx.reset_kernel_timing()
        check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), 8, 1, 256, 0.7, 2,
                               C.byref(out), 0))
        res.append({k: ctx.kernel_time(k)[0] for k in ("group_eval", "fast_build", "group_table")})
    ge = min(x["group_eval"] for x in res)
    base = base or ge
    print(f"c={c} S={S}: group_eval {ge:.3f} ms (rel {ge / base:.3f}), fast_build "
          f"{min(x['fast_build'] for x in res):.3f} ms, group_table {min(x['group_table'] for x in res):.3f} ms")
