"""GPU parity for the Monte-Carlo scaling sweep (C4): device scenario
generation, per (scenario, candidate) t_total / cost bit-exact, n_star exact,
aggregates consistent."""
import ctypes as C

import numpy as np
import pytest

from cases import c4_spec, profiles
from oracle_lib import port
from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.lib import check, context, ptr
from paper_2602_22718_b200.rollsim import default_profile

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def rs_generate(spec):
    ctx = context()
    n = spec.n_scenarios * spec.count
    pred = np.zeros(n, np.float64)
    plen = np.zeros(n, np.int32)
    check(ctx.lib.rs_generate_scenarios(ctx.handle, C.byref(spec), pred.ctypes.data_as(C.c_void_p),
                                        plen.ctypes.data_as(C.c_void_p), 0))
    return pred, plen


def rs_sweep(spec, prof, g, n_min, n_max, lam, gpus, arrays=None):
    ctx = context()
    S, Cn = spec.n_scenarios, n_max - n_min + 1
    out = {"t_total": np.zeros(S * Cn), "cost": np.zeros(S * Cn),
           "idle": np.zeros(S * Cn, np.int64), "n_star": np.zeros(S, np.int32),
           "hist": np.zeros(Cn, np.int32), "sum_t": np.zeros(Cn), "sum_c": np.zeros(Cn)}
    so = _abi.RsSweepOut(*[out[k].ctypes.data for k in
                           ("t_total", "cost", "idle", "n_star", "hist", "sum_t", "sum_c")])
    s, keep = prof.struct()
    if arrays is None:
        check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(s), g, n_min, n_max, lam, gpus,
                               C.byref(so), 0))
    else:
        pred, plen = arrays
        check(ctx.lib.rs_sweep_arrays(ctx.handle, pred.ctypes.data, plen.ctypes.data, S,
                                      spec.count, C.byref(s), g, n_min, n_max, lam, gpus,
                                      C.byref(so), 0))
    out["t_total"] = out["t_total"].reshape(S, Cn)
    out["cost"] = out["cost"].reshape(S, Cn)
    out["idle"] = out["idle"].reshape(S, Cn)
    return out


def test_generator_matches_oracle():
    spec = c4_spec(3, count=20000, first=17)
    p1, l1 = rs_generate(spec)
    p2, l2 = port().generate_scenarios(spec)
    assert np.array_equal(bits(p1), bits(p2)) and np.array_equal(l1, l2)
    assert p1.min() >= 1.0 and p1.max() <= 16384.0 and (p1 == 16384.0).any()


def check_sweep(spec, n_min, n_max, prof=None, lam=0.7, g=8, arrays=False):
    prof = prof or default_profile()
    pred, plen = port().generate_scenarios(spec)
    got = rs_sweep(spec, prof, g, n_min, n_max, lam, 2, (pred, plen) if arrays else None)
    S, P = spec.n_scenarios, spec.count
    tt, cc, ns = port().sweep_arrays(pred, plen, S, P, prof, g, n_min, n_max, lam, 2, threads=8)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(bits(got["cost"]), bits(cc))
    assert np.array_equal(got["n_star"], ns)
    for s in range(S):
        idle = port().scale_idle(pred[s * P:(s + 1) * P], None, g, n_min, n_max)
        assert np.array_equal(got["idle"][s], idle)
    hist = np.bincount(ns - n_min, minlength=n_max - n_min + 1)
    assert np.array_equal(got["hist"], hist)
    np.testing.assert_allclose(got["sum_t"], tt.sum(axis=0), rtol=1e-12)
    np.testing.assert_allclose(got["sum_c"], cc.sum(axis=0), rtol=1e-12)
    return got


def test_sweep_small_bitwise():
    check_sweep(c4_spec(12, count=3000, first=5), 1, 64)


def test_sweep_multi_batch_host_outputs():
    """More scenarios than one batch holds (<= 2,048): each batch's host
    results leave on the copy stream while the next batch computes, through
    two alternating buffer sets; every batch must land intact."""
    check_sweep(c4_spec(4200, count=64, first=31), 1, 24)


def test_sweep_arrays_bitwise_and_nmin():
    check_sweep(c4_spec(5, count=2048, first=100), 3, 50, arrays=True, lam=0.3, g=4)


def test_sweep_other_profiles():
    for name in ("small", "constant"):
        check_sweep(c4_spec(3, count=1024, first=9), 1, 32, prof=profiles()[name], lam=1.0)


def test_sweep_unbounded_arrays_generic_path():
    spec = c4_spec(3, count=1500, first=1)
    pred, plen = port().generate_scenarios(spec)
    pred = pred * 7.0  # pushes finish ticks past the bucketed range
    got = rs_sweep(spec, default_profile(), 8, 1, 40, 0.7, 2, (pred, plen))
    tt, cc, ns = port().sweep_arrays(pred, plen, 3, 1500, default_profile(), 8, 1, 40, 0.7, 2)
    assert np.array_equal(bits(got["t_total"]), bits(tt)) and np.array_equal(got["n_star"], ns)


@pytest.mark.slow
def test_sweep_full_size_scenarios_bitwise():
    """C4 at full scenario size: 65,536 prompts x G=8, N in [1, 256]."""
    check_sweep(c4_spec(2, count=65536, first=4242), 1, 256)


def test_sweep_select_matches_oracle():
    rng = np.random.RandomState(0)
    st, sc = rng.rand(64) * 100, rng.rand(64) * 3
    ctx = context()
    ns = C.c_int32()
    check(ctx.lib.rs_sweep_select(ptr(st, C.c_double), ptr(sc, C.c_double), 1000, 64, 1, 0.7,
                                  C.byref(ns)))
    assert ns.value == port().sweep_select(st, sc, 1000, 1, 0.7)


def test_sweep_many_scenarios_lockstep_bitwise():
    """S >= #SMs takes the candidate-lockstep evaluator."""
    check_sweep(c4_spec(160, count=2048, first=77), 1, 96)


def test_sweep_many_scenarios_other_profile_lockstep():
    check_sweep(c4_spec(150, count=1500, first=5), 2, 70, prof=profiles()["small"], g=3, lam=0.4)


def test_sweep_wide_buckets_bitwise():
    """Buckets wider than a shared-memory window (~3,000 equal finish ticks,
    ranked in global memory) and wider than the fast path allows (> 4,096,
    generic path), with duplicate predictions tie-broken by id."""
    rng = np.random.RandomState(21)
    S, P = 3, 9000
    pred = rng.uniform(1.0, 3000.0, S * P)
    plen = rng.randint(0, 2000, S * P).astype(np.int32)
    pred[0:3000] = 512.0                                   # scenario 0: one 3,000-wide bucket
    pred[P:P + 2000] = 7.25
    pred[P + 2000:P + 3500] = rng.uniform(99.0, 100.0, 1500)  # scenario 1: two wide buckets
    pred[2 * P:2 * P + 5000] = 40.0                        # scenario 2: > 4,096 -> generic path
    spec = c4_spec(S, count=P)
    got = rs_sweep(spec, default_profile(), 8, 1, 64, 0.6, 2, (pred, plen))
    tt, cc, ns = port().sweep_arrays(pred, plen, S, P, default_profile(), 8, 1, 64, 0.6, 2,
                                     threads=3)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(bits(got["cost"]), bits(cc))
    assert np.array_equal(got["n_star"], ns)


def test_sweep_lockstep_wide_candidate_range():
    """More than 256 candidates: two lockstep CTAs per scenario, select and
    aggregate unfused (S >= 32 takes the lockstep evaluator)."""
    check_sweep(c4_spec(40, count=1400, first=321), 2, 320, lam=0.55, g=4)


def test_sweep_lockstep_wide_batch_profile():
    """Lockstep evaluator with a large batch axis (G=1, batch knots to 2,048:
    2,047 small-batch rows, a 2,048-entry clamped tail) and fractional context
    knots (piece ends from floor/ceil of non-integers)."""
    from paper_2602_22718_b200.rollsim import LatencyProfile
    bk = [1.0, 7.5, 64.0, 512.0, 2048.0]
    ck = [50.0, 333.3, 1500.5, 3000.0]
    grid = [[0.004 + 1e-5 * b + 2e-6 * c + 3e-9 * b * c for c in ck] for b in bk]
    prof = LatencyProfile(bk, ck, grid, 0.0007, 2)
    check_sweep(c4_spec(40, count=1000, first=888), 1, 64, prof=prof, lam=0.35, g=1)


def test_sweep_huge_batch_axis_falls_back():
    """A batch axis too long for the lockstep evaluator's shared-memory tail
    (G=1, batch knots to 32,768) takes the per-group evaluator, same bits."""
    from paper_2602_22718_b200.rollsim import LatencyProfile
    bk = [1.0, 1024.0, 32768.0]
    ck = [128.0, 4096.0]
    grid = [[0.005 + 1e-6 * b + 1e-6 * c for c in ck] for b in bk]
    prof = LatencyProfile(bk, ck, grid, 0.0005, 2)
    check_sweep(c4_spec(36, count=600, first=5), 1, 40, prof=prof, lam=0.5, g=1)


def test_sweep_generated_wide_bucket_falls_back():
    """a generated spec whose clamp puts > 4,096 prompts
    into one finish bucket (pred_max = 2,048: ~24 % of 65,536 prompts) must
    not reuse stale structure data: the fast build flags it, the kernels that
    read the structure skip, and the sweep reruns on the generic path."""
    spec = c4_spec(3, count=65536, first=11)
    spec.pred_max = 2048.0
    check_sweep(spec, 1, 48)


def test_sweep_late_wide_bucket_reruns_generic():
    """Several batches of caller arrays (host inputs streamed on in_stream),
    the LAST scenario holding a bucket wider than the fast path takes: the
    end-of-sweep status check reruns everything on the generic path."""
    spec = c4_spec(2300, count=600, first=3)
    pred, plen = port().generate_scenarios(spec)
    pred[-600:] = 77.0
    pred[-5000:-4700] = 12.5
    got = rs_sweep(spec, default_profile(), 8, 1, 16, 0.7, 2, (pred, plen))
    tt, cc, ns = port().sweep_arrays(pred, plen, 2300, 600, default_profile(), 8, 1, 16, 0.7, 2,
                                     threads=8)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(bits(got["cost"]), bits(cc))
    assert np.array_equal(got["n_star"], ns)


def test_sweep_first_batch_too_wide_reruns_generic():
    """The same with the wide bucket in the first batch (caught by the early
    status check after batch 0) — and > 4,096 equal predictions."""
    spec = c4_spec(2200, count=4200, first=8)
    pred, plen = port().generate_scenarios(spec)
    pred[:4200] = 333.0
    got = rs_sweep(spec, default_profile(), 8, 1, 8, 0.7, 2, (pred, plen))
    tt, cc, ns = port().sweep_arrays(pred, plen, 2200, 4200, default_profile(), 8, 1, 8, 0.7, 2,
                                     threads=8)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(got["n_star"], ns)


def test_sweep_arrays_multi_batch_streamed_inputs():
    """Caller arrays over several batches: batch i+1's inputs are copied on
    the input stream while batch i computes (two input sets)."""
    check_sweep(c4_spec(4300, count=96, first=57), 1, 20, arrays=True, lam=0.45)


def test_sweep_multi_batch_pinned_outputs():
    """Pinned caller outputs take the direct (no bounce) copy path."""
    import torch
    spec = c4_spec(4200, count=64, first=31)
    S, Cn = spec.n_scenarios, 24
    prof = default_profile()
    ctx = context()
    t = {k: torch.zeros(n, dtype=d).pin_memory() for k, n, d in
         (("t_total", S * Cn, torch.float64), ("cost", S * Cn, torch.float64),
          ("idle", S * Cn, torch.int64), ("n_star", S, torch.int32))}
    so = _abi.RsSweepOut(t["t_total"].data_ptr(), t["cost"].data_ptr(), t["idle"].data_ptr(),
                         t["n_star"].data_ptr(), None, None, None)
    s, keep = prof.struct()
    check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(s), 8, 1, Cn, 0.7, 2, C.byref(so), 0))
    pred, plen = port().generate_scenarios(spec)
    tt, cc, ns = port().sweep_arrays(pred, plen, S, 64, prof, 8, 1, Cn, 0.7, 2, threads=8)
    assert np.array_equal(bits(t["t_total"].numpy().reshape(S, Cn)), bits(tt))
    assert np.array_equal(bits(t["cost"].numpy().reshape(S, Cn)), bits(cc))
    assert np.array_equal(t["n_star"].numpy(), ns)


def test_sweep_evaluator_thresholds_bitwise():
    """Both sides of the small-batch evaluator's thresholds (fast_eval with
    every group per warp up to 8 scenarios, N < 128 per warp above, the
    lockstep walk from 56): same bits as the oracle, candidates past 128."""
    for S in (8, 9, 55, 56):
        check_sweep(c4_spec(S, count=4096, first=300 + S), 1, 160)
