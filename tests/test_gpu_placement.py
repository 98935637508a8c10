"""GPU parity for scale() with plan_rlhfless's placement penalty
(proj/src/training.cpp:150-164) computed on the device (rs_scale_placed):
per-candidate penalties, totals, scores and N* bitwise against the reference
(oracle/_ref) when it is built, else against the C restatement."""
import ctypes as C

import numpy as np
import pytest

from cases import Rng, c4_spec, placement_cases, random_predicted, small_profile
from oracle_lib import port, ref
from paper_2602_22718_b200 import _abi, rollsim
from paper_2602_22718_b200.lib import ConfigError, PlacementError, ValidationError, check, context, ptr
from paper_2602_22718_b200.rollsim import (ClusterTopology, PlacementPenalty, PredictedPrompt,
                                           default_profile, default_topology)

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def oracle():
    return ref() or port()


def rs_scale_placed(pred, plen, rank, prof, g, n_min, n_max, lam, gpus, pen):
    ctx = context()
    P = len(pred)
    Cn = n_max - n_min + 1
    arr = {k: np.zeros(Cn) for k in ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score")}
    order = np.zeros(P, np.int32)
    out = _abi.RsScaleOut(0, *[ptr(arr[k], C.c_double) for k in
                               ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score")],
                          None, ptr(order, C.c_int32), None, None)
    s, keep = prof.struct()
    pp, keep_p = pen.struct()
    check(ctx.lib.rs_scale_placed(ctx.handle, ptr(np.ascontiguousarray(pred, np.float64), C.c_double),
                                  ptr(np.ascontiguousarray(plen, np.int32), C.c_int32),
                                  ptr(rank, C.c_int32) if rank is not None else None, P,
                                  C.byref(s), g, n_min, n_max, float(lam), gpus, C.byref(pp),
                                  C.byref(out)))
    arr.update(n_star=out.n_star, order=order)
    return arr


def same(a, b, ctx):
    assert a["n_star"] == b["n_star"], ctx
    for k in ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score"):
        assert np.array_equal(bits(a[k]), bits(b[k])), (ctx, k)
    assert a["order"].tolist() == b["order"].tolist(), ctx


def test_placement_penalty_random_bitwise():
    rng = Rng(515)
    for ci, (pen, gpus, cap) in enumerate(placement_cases()):
        for trial in range(6):
            count = rng.uniform_int(cap, 60)
            pred, plen = random_predicted(rng, count, 1.0, 900.0, 1, 900, integer=trial % 2 == 0)
            rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
            prof = [default_profile(), small_profile()][trial % 2]
            n_max = min(cap, count)
            got = rs_scale_placed(pred, plen, rank, prof, 4, 1, n_max, 0.6, gpus, pen)
            want = oracle().scale_placed(pred, plen, rank, prof, 4, 1, n_max, 0.6, gpus, pen)
            same(got, want, (ci, trial))
            assert (got["t_penalty"] >= 0).all()


def test_placement_penalty_c3_shape():
    """C3: one 65,536-prompt scenario over N in [1, 512] on
    default_topology(128, 8, 4) (1,024 GPUs, up to 512 actors of 2 GPUs). The
    decode tail (~960 s, the 16,384-token clamp) dwarfs realistic transfers, so
    the model size is inflated to make the penalty bind for ~1/4 of the N."""
    pred, plen = port().generate_scenarios(c4_spec(1, count=65536, first=3))
    pen = PlacementPenalty(default_topology(128, 8, 4), l_prefill_seconds=0.3, model_bytes=1e12)
    got = rs_scale_placed(pred, plen, None, default_profile(), 8, 1, 512, 0.7, 2, pen)
    want = port().scale_placed(pred, plen, None, default_profile(), 8, 1, 512, 0.7, 2, pen)
    same(got, want, "c3")
    assert (got["t_penalty"] > 0).any()


def test_placement_penalty_through_mirror_api():
    rng = Rng(9)
    pred, plen = random_predicted(rng, 48, 1.0, 600.0, 1, 600)
    predicted = [PredictedPrompt(f"p{i:06d}", int(plen[i]), float(pred[i])) for i in range(48)]
    pen = placement_cases()[2][0]
    res = rollsim.scale(predicted, default_profile(), 4, 1, 12, 0.6, 2, penalty=pen)
    want = oracle().scale_placed(pred, plen, None, default_profile(), 4, 1, 12, 0.6, 2, pen)
    assert res.n_star == want["n_star"]
    assert [c.t_penalty for c in res.candidates] == want["t_penalty"].tolist()
    assert [c.score for c in res.candidates] == want["score"].tolist()


def test_placement_penalty_errors():
    pred, plen = random_predicted(Rng(3), 40)
    predicted = [PredictedPrompt(f"p{i:06d}", int(plen[i]), float(pred[i])) for i in range(40)]
    pen, gpus, cap = placement_cases()[0]
    with pytest.raises(PlacementError):
        rollsim.scale(predicted, default_profile(), 2, 1, cap + 1, 0.5, gpus, penalty=pen)
    bad = PlacementPenalty(ClusterTopology([8, 8], intra_node_bw=1e9, inter_node_bw=2e9),
                           l_prefill_seconds=0.1)
    with pytest.raises(ConfigError):
        rollsim.scale(predicted, default_profile(), 2, 1, 4, 0.5, gpus, penalty=bad)
    with pytest.raises(ValidationError):  # scale's own checks come first
        rollsim.scale(predicted, default_profile(), 2, 1, 41, 0.5, gpus, penalty=bad)
    neg = PlacementPenalty(default_topology(2, 8, 4), l_prefill_seconds=0.1, model_bytes=-1.0)
    with pytest.raises(ConfigError):
        rollsim.scale(predicted, default_profile(), 2, 1, 4, 0.5, gpus, penalty=neg)
