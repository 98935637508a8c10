import ctypes as C, sys, pathlib
REPO = pathlib.Path("/root/repo"); sys.path[:0] = [str(REPO), str(REPO / "tests")]
import torch, numpy as np
from cases import c4_spec
from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.lib import check, context
from paper_2602_22718_b200.rollsim import default_profile
ctx = context(0); ps, keep = default_profile().struct()
S = 1184; spec = c4_spec(S, count=65536)
pred = torch.empty(S * 65536, dtype=torch.float64, device="cuda"); plen = torch.empty(S * 65536, dtype=torch.int32, device="cuda")
check(ctx.lib.rs_generate_scenarios(ctx.handle, C.byref(spec), C.c_void_p(pred.data_ptr()), C.c_void_p(plen.data_ptr()), 1))
torch.cuda.synchronize()
o = [torch.empty(S * 256, dtype=torch.float64, device="cuda") for _ in range(2)]; ns = torch.empty(S, dtype=torch.int32, device="cuda")
out = _abi.RsSweepOut(o[0].data_ptr(), o[1].data_ptr(), None, ns.data_ptr(), None, None, None)
ctx.enable_kernel_timing(True)
for r in range(3):
    ctx.reset_kernel_timing()
    check(ctx.lib.rs_sweep_arrays(ctx.handle, C.c_void_p(pred.data_ptr()), C.c_void_p(plen.data_ptr()), S, 65536, C.byref(ps), 8, 1, 256, 0.7, 2, C.byref(out), 1))
    print(r, {k: round(ctx.kernel_time(k)[0], 3) for k in ("validate_inputs", "fast_build", "group_table", "group_eval", "finish")})
ctx.reset_kernel_timing()
check(ctx.lib.rs_generate_scenarios(ctx.handle, C.byref(spec), C.c_void_p(pred.data_ptr()), C.c_void_p(plen.data_ptr()), 1))
torch.cuda.synchronize(); ctx.synchronize()
print("gen", ctx.kernel_time("gen_scenarios"))
