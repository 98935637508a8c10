"""Time the C2 prefix-index build (device-resident and host CSR) per kernel."""
import ctypes as C
import pathlib
import sys
import time

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cases import c2_tokens  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402

tok, off = c2_tokens()
ctx = context(0)
d_tok = torch.from_numpy(tok).cuda()
d_off = torch.from_numpy(off).cuda()
lib = ctx.lib
h = C.c_void_p()
names = ["dedup_init", "dedup_compare_r0", "dedup_refine", "dedup_compare",
         "dedup_finalize", "dedup_compact", "dedup_tables"]
for rep in range(4):
    ctx.enable_kernel_timing(True)
    ctx.reset_kernel_timing()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    check(lib.rs_prefix_index_build_device(ctx.handle, C.c_void_p(d_tok.data_ptr()),
                                           C.c_void_p(d_off.data_ptr()), len(off) - 1, C.byref(h)))
    dt = time.perf_counter() - t0
    lib.rs_prefix_index_free(h)
    print(f"rep {rep}: device build {dt * 1e3:.3f} ms")
    if rep == 3:
        for n in names:
            ms, k = ctx.kernel_time(n)
            print(f"   {n:20s} {ms:8.3f} ms over {k} launches")
pt = torch.from_numpy(tok).pin_memory()
po = torch.from_numpy(off).pin_memory()
for rep in range(3):
    t0 = time.perf_counter()
    check(lib.rs_prefix_index_build(ctx.handle, pt.numpy().ctypes.data_as(C.POINTER(C.c_int32)),
                                    po.numpy().ctypes.data_as(C.POINTER(C.c_int64)), len(off) - 1,
                                    C.byref(h)))
    print(f"host build {1e3 * (time.perf_counter() - t0):.1f} ms")
    lib.rs_prefix_index_free(h)
t0 = time.perf_counter()
x = torch.empty_like(pt, device="cuda")
torch.cuda.synchronize()
t0 = time.perf_counter()
x.copy_(pt, non_blocking=True)
torch.cuda.synchronize()
print(f"torch pinned H2D of {pt.numel() * 4 / 1e6:.0f} MB: {1e3 * (time.perf_counter() - t0):.1f} ms")
