"""Multi-GPU Monte-Carlo scaling sweep.

Scenarios are independent: rank r of W evaluates the contiguous block
shard_range(S, W, r) on its own GPU (rs_sweep, device-resident outputs).
The only exchange is one all-reduce of the per-candidate aggregates
(sum of t_total, sum of cost, n_star histogram: ~5 KB), after which every
rank picks the aggregate N* with rs_sweep_select (mean t / mean cost,
min-max normalised like scale(), first strict minimum).
"""
import ctypes as C

import numpy as np

from . import _abi
from .lib import as_f64, check, load, ptr


def shard_range(n_scenarios, world, rank):
    """Contiguous block of scenarios owned by `rank` (sizes differ by <= 1)."""
    return n_scenarios * rank // world, n_scenarios * (rank + 1) // world


def combine(sum_t, sum_c, hist, group=None):
    """All-reduce (SUM) of the per-candidate aggregates, in place.
    Tensors may live on the GPU (NCCL) or the CPU (gloo)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return sum_t, sum_c, hist
    dist.all_reduce(sum_t, group=group)
    dist.all_reduce(sum_c, group=group)
    dist.all_reduce(hist, group=group)
    return sum_t, sum_c, hist


def aggregate_pick(sum_t, sum_c, n_scenarios, n_min, lam):
    """N* of the whole sweep from the combined aggregates (host, O(C))."""
    st, sc = as_f64(sum_t), as_f64(sum_c)
    ns = C.c_int32()
    check(load().rs_sweep_select(ptr(st, C.c_double), ptr(sc, C.c_double), int(n_scenarios),
                                 len(st), n_min, float(lam), C.byref(ns)))
    return ns.value


def sweep_device(ctx, spec, profile, G, n_min, n_max, lam, gpus_per_actor, out_tensors):
    """rs_sweep with device outputs (torch CUDA tensors: t_total, cost, idle,
    n_star, hist, sum_t, sum_c); asynchronous on the context stream."""
    ps, keep = profile.struct()
    ts = [out_tensors[k] for k in ("t_total", "cost", "idle", "n_star", "hist", "sum_t", "sum_c")]
    so = _abi.RsSweepOut(*[t.data_ptr() if t is not None else None for t in ts])
    check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(ps), G, n_min, n_max, float(lam),
                           gpus_per_actor, C.byref(so), 1))
    return out_tensors
