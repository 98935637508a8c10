"""dedup_tables into device memory (rs_prefix_index_build_device_async) vs
into mapped pinned host memory (rs_prefix_index_build_device): CUDA-event
time of the tables kernel, C2 batch."""
import ctypes as C
import pathlib
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import torch  # noqa: E402
from cases import c2_tokens  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402

tok, off = c2_tokens()
ctx = context(0)
d_tok = torch.from_numpy(tok).cuda()
d_off = torch.from_numpy(off).cuda()
lib = ctx.lib
tabs = torch.empty(5 * 2562, dtype=torch.int64, device="cuda")
info = torch.empty(5, dtype=torch.int64, device="cuda")
h = C.c_void_p()
for mode in ("mapped", "device"):
    ctx.enable_kernel_timing(True)
    for rep in range(25):
        if rep == 5:
            ctx.reset_kernel_timing()
        if mode == "mapped":
            check(lib.rs_prefix_index_build_device(ctx.handle, C.c_void_p(d_tok.data_ptr()),
                                                   C.c_void_p(d_off.data_ptr()), len(off) - 1, C.byref(h)))
            lib.rs_prefix_index_free(h)
        else:
            check(lib.rs_prefix_index_build_device_async(ctx.handle, C.c_void_p(d_tok.data_ptr()),
                                                         C.c_void_p(d_off.data_ptr()), len(off) - 1, 2560,
                                                         C.c_void_p(tabs.data_ptr()), C.c_void_p(info.data_ptr())))
            ctx.synchronize()
    ms, n = ctx.kernel_time("dedup_tables")
    print(mode, f"tables {1e3 * ms / n:.1f} us", {k: round(1e3 * ctx.kernel_time(k)[0] / max(ctx.kernel_time(k)[1], 1), 1)
                                                  for k in ("dedup_init", "dedup_compare_r0", "dedup_refine")})
