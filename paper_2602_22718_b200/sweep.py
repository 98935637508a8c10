"""Multi-GPU Monte-Carlo scaling sweep.

Scenarios are independent: rank r of W evaluates the contiguous block
shard_range(S, W, r) on its own GPU. The only exchange is ONE all-reduce of
the packed per-candidate aggregates (sum of t_total, sum of cost, n_star
histogram as FP64: 3 x C doubles, ~6 KB), after which every rank picks the
aggregate N* (mean t / mean cost, min-max normalised like scale(), first
strict minimum).

On the GPU the exchange lives inside librs_b200 (`Comm` + rs_sweep_sharded:
NCCL over NVLink, the library's own communicator); `combine` is the same
packed exchange over a torch.distributed group (gloo on CPU in the tests).
"""
import ctypes as C

import numpy as np

from .lib import as_f64, check, load, ptr


def shard_range(n_scenarios, world, rank):
    """Contiguous block of scenarios owned by `rank` (sizes differ by <= 1);
    the same split rs_sweep_sharded uses."""
    return n_scenarios * rank // world, n_scenarios * (rank + 1) // world


def combine(sum_t, sum_c, hist, group=None):
    """One all-reduce (SUM) of the packed aggregates, results written back in
    place. Tensors may live on the GPU (NCCL) or the CPU (gloo)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return sum_t, sum_c, hist
    pack = torch.cat([sum_t.to(torch.float64), sum_c.to(torch.float64), hist.to(torch.float64)])
    dist.all_reduce(pack, group=group)
    n = sum_t.numel()
    sum_t.copy_(pack[:n])
    sum_c.copy_(pack[n:2 * n])
    hist.copy_(pack[2 * n:].round().to(hist.dtype))
    return sum_t, sum_c, hist


def aggregate_pick(sum_t, sum_c, n_scenarios, n_min, lam):
    """N* of the whole sweep from the combined aggregates (host, O(C))."""
    st, sc = as_f64(sum_t), as_f64(sum_c)
    ns = C.c_int32()
    check(load().rs_sweep_select(ptr(st, C.c_double), ptr(sc, C.c_double), int(n_scenarios),
                                 len(st), n_min, float(lam), C.byref(ns)))
    return ns.value


class Comm:
    """librs_b200's NCCL communicator for rs_sweep_sharded (one per rank).
    The 128-byte id is made on rank 0 and shipped with `broadcast`, a
    callable (bytes on rank 0 -> bytes on every rank), e.g. over
    torch.distributed.broadcast_object_list."""

    def __init__(self, ctx, world, rank, broadcast):
        lib = load()
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            check(lib.rs_comm_unique_id(uid))
        uid = (C.c_uint8 * 128).from_buffer_copy(broadcast(bytes(uid)))
        h = C.c_void_p()
        check(lib.rs_comm_init(ctx.handle, uid, world, rank, C.byref(h)))
        self.handle, self.lib, self.world, self.rank = h, lib, world, rank

    def close(self):
        if self.handle:
            self.lib.rs_comm_destroy(self.handle)
            self.handle = None


class Multi:
    """rs_multi: one process driving several GPUs (a context per device and
    an NCCL clique), e.g. for `rs_multi_sweep` over host outputs."""

    def __init__(self, devices):
        lib = load()
        d = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        check(lib.rs_multi_create(ptr(d, C.c_int32), len(d), C.byref(h)))
        self.handle, self.lib, self.n = h, lib, len(d)

    def close(self):
        if self.handle:
            self.lib.rs_multi_destroy(self.handle)
            self.handle = None
