"""Where the C2 device build's wall time goes: host wall clock per call vs
GPU time between events recorded on the context stream around the call,
and the per-kernel CUDA-event times (50 calls each)."""
import ctypes as C
import pathlib
import sys
import time

REPO = pathlib.Path(__file__).resolve().parents[1]
sys.path[:0] = [str(REPO), str(REPO / "tests")]
import torch  # noqa: E402
from cases import c2_tokens  # noqa: E402
from paper_2602_22718_b200.lib import check, context  # noqa: E402

tok, off = c2_tokens()
ctx = context(0)
s = torch.cuda.Stream()
ctx.set_stream(s.cuda_stream)
d_tok = torch.from_numpy(tok).cuda()
d_off = torch.from_numpy(off).cuda()
lib = ctx.lib
h = C.c_void_p()


def build():
    check(lib.rs_prefix_index_build_device(ctx.handle, C.c_void_p(d_tok.data_ptr()),
                                           C.c_void_p(d_off.data_ptr()), len(off) - 1, C.byref(h)))
    lib.rs_prefix_index_free(h)


for _ in range(5):
    build()
n = 50
walls, gpus = [], []
for _ in range(n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0.record(s)
    build()
    e1.record(s)
    e1.synchronize()
    walls.append(time.perf_counter() - t0)
    gpus.append(e0.elapsed_time(e1))
walls.sort()
gpus.sort()
print(f"wall median {1e3 * walls[n // 2]:.3f} ms, GPU (events) median {gpus[n // 2]:.3f} ms")
ctx.enable_kernel_timing(True)
ctx.reset_kernel_timing()
for _ in range(n):
    build()
tot = 0
for k in ("dedup_init", "dedup_compare_r0", "dedup_refine", "dedup_tables"):
    ms, cnt = ctx.kernel_time(k)
    tot += ms / max(cnt, 1)
    print(f"  {k:18s} {1e3 * ms / max(cnt, 1):8.1f} us")
print(f"  kernels sum {1e3 * tot:.1f} us")
