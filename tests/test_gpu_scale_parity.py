"""Bit-exactness at the headline scale and in the regimes round 1 left
untested ("Next round" item 1):

- a full-size C4 batch (65,536 prompts x G=8, N in [1, 256]) of more than
  one wave through the lockstep evaluator, every scenario checked bitwise;
- LPT at the C3 configuration (65,536 x 8 rollouts onto N in {1, 2, 7, 64,
  255, 512} actors) against orc_lpt;
- the dedup map and block hashes at C2 size;
- the C2 variant with 8 system prompts;
- a sweep under a long-context profile (context knots to 32,768), which
  takes the warp-cooperative evaluator from global memory.
All against the C port (oracle/rs_oracle.c), itself pinned to the reference.
"""
import ctypes as C
import time

import numpy as np
import pytest

import paper_2602_22718_b200.rollsim as rs
from cases import c2_tokens, c2_tokens_multi, c4_spec, long_context_profile
from oracle_lib import port, ref
from paper_2602_22718_b200 import _abi
from paper_2602_22718_b200.lib import check, context
from paper_2602_22718_b200.rollsim import PrefixIndex, default_profile

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def sweep(spec, prof, g, n_min, n_max, lam, gpus=2):
    ctx = context()
    S, Cn = spec.n_scenarios, n_max - n_min + 1
    out = {"t_total": np.zeros(S * Cn), "cost": np.zeros(S * Cn),
           "idle": np.zeros(S * Cn, np.int64), "n_star": np.zeros(S, np.int32),
           "hist": np.zeros(Cn, np.int32), "sum_t": np.zeros(Cn), "sum_c": np.zeros(Cn)}
    so = _abi.RsSweepOut(*[out[k].ctypes.data for k in
                           ("t_total", "cost", "idle", "n_star", "hist", "sum_t", "sum_c")])
    s, keep = prof.struct()
    t0 = time.perf_counter()
    check(ctx.lib.rs_sweep(ctx.handle, C.byref(spec), C.byref(s), g, n_min, n_max, lam, gpus,
                           C.byref(so), 0))
    out["seconds"] = time.perf_counter() - t0
    for k in ("t_total", "cost", "idle"):
        out[k] = out[k].reshape(S, Cn)
    return out


@pytest.mark.slow
def test_c4_full_size_lockstep_batch_bitwise():
    """600 full-size C4 scenarios: more than one wave of the lockstep
    evaluator (4 CTAs x 148 SMs = 592 slots), every scenario bitwise
    (t_total, cost, n_star), idle slot-ticks on every 10th."""
    S, P = 600, 65536
    spec = c4_spec(S, count=P, first=5000)
    got = sweep(spec, default_profile(), 8, 1, 256, 0.7)
    pred, plen = port().generate_scenarios(spec)
    tt, cc, ns = port().sweep_arrays(pred, plen, S, P, default_profile(), 8, 1, 256, 0.7, 2,
                                     threads=16)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(bits(got["cost"]), bits(cc))
    assert np.array_equal(got["n_star"], ns)
    for s in range(0, S, 10):
        assert np.array_equal(got["idle"][s], port().scale_idle(pred[s * P:(s + 1) * P], None,
                                                                8, 1, 256)), s


@pytest.mark.slow
def test_lpt_at_c3():
    """C3: 65,536 prompts x G=8 = 524,288 rollouts (lognormal lengths to
    16,384) onto N actors, makespan and idle exact against orc_lpt."""
    pred, _ = port().generate_scenarios(c4_spec(1, count=65536, first=0))
    rank = np.random.RandomState(5).permutation(65536).astype(np.int32)
    for n in (1, 2, 7, 64, 255, 512):
        mk, idle = rs.lpt(pred, rank, 8, n, n)
        wmk, widle = port().lpt(pred, rank, 8, n, n)
        assert (mk.tolist(), idle.tolist()) == (wmk.tolist(), widle.tolist()), n
    # a candidate range in one call (one warp per N)
    mk, idle = rs.lpt(pred, rank, 8, 250, 260)
    wmk, widle = port().lpt(pred, rank, 8, 250, 260)
    assert mk.tolist() == wmk.tolist() and idle.tolist() == widle.tolist()


@pytest.mark.slow
def test_dedup_map_and_block_hashes_at_c2():
    tok, off = c2_tokens()
    for l in (1, 2048, 2049, 2050, 2560):
        got = rs.dedup_map((tok, off), l)
        want = port().dedup_map(tok, off, l)
        assert np.array_equal(got, want), l
        assert rs.unique_prefix_count_among((tok, off), l) == len(np.unique(want))
    assert rs.dedup_map((tok, off), 2048).max() == 0  # one shared system prompt
    for k in (16, 128):
        assert np.array_equal(rs.block_hashes((tok, off), k), port().block_hashes(tok, off, k)), k


@pytest.mark.slow
def test_c2_eight_system_prompts():
    """SURVEY §8d's C2 variant: 8 distinct 2,048-token system prompts."""
    tok, off = c2_tokens_multi(n_sys=8)
    idx = PrefixIndex.build((tok, off))
    _, want = port().prefix_tables(tok, off)
    for a, b in zip(idx.tables(), want):
        assert a.tolist() == b.tolist()
    assert idx.unique_prefix_count(2048) == 8
    R = ref()
    if R is not None:  # the reference itself, on the same batch
        info, u, t, r = R.prefix_curves(tok, off, 2562)
        assert [idx.unique_prefix_count(l) for l in range(1, 2563)] == u.tolist()
        assert [idx.remainder_tokens(l) for l in range(1, 2563)] == r.tolist()
    sel = rs.select_prefix_length(idx, rs.PrefillCapacity(64), 1, idx.max_prompt_len())
    assert sel.prefix_len == 2048 and not sel.capacity_exceeded
    got = rs.dedup_map((tok, off), 2048)
    assert got.tolist() == (np.arange(65536) % 8).tolist()
    assert np.array_equal(got, port().dedup_map(tok, off, 2048))


@pytest.mark.parametrize("S,P", [(3, 65536), (40, 8192)])
def test_sweep_long_context_profile(S, P):
    """Context knots to 32,768 (a 32,641-entry context memo): the sweep
    runs every group warp-cooperatively from global memory; bitwise."""
    prof = long_context_profile()
    spec = c4_spec(S, count=P, first=31)
    got = sweep(spec, prof, 8, 1, 64, 0.6)
    pred, plen = port().generate_scenarios(spec)
    tt, cc, ns = port().sweep_arrays(pred, plen, S, P, prof, 8, 1, 64, 0.6, 2, threads=8)
    assert np.array_equal(bits(got["t_total"]), bits(tt))
    assert np.array_equal(bits(got["cost"]), bits(cc))
    assert np.array_equal(got["n_star"], ns)
    print(f"long-context sweep S={S} P={P}: {got['seconds'] * 1e3:.1f} ms "
          f"({S * 64 / got['seconds']:.0f} evals/s)")


def test_scale_with_lpt_outputs():
    """scale() with the LPT extension's outputs (rs_scale_out.lpt_makespan /
    lpt_idle): per candidate equal to orc_lpt on the same predictions, and
    the scale() results themselves unchanged (bitwise vs the port)."""
    pred, plen = port().generate_scenarios(c4_spec(1, count=4096, first=77))
    ps = [rs.PredictedPrompt(f"p{i:06d}", int(plen[i]), float(pred[i])) for i in range(len(pred))]
    got = rs.scale(ps, default_profile(), 8, 1, 64, 0.7, 2, with_lpt=True)
    wmk, widle = port().lpt(pred, None, 8, 1, 64)
    assert got.lpt_makespan.tolist() == wmk.tolist()
    assert got.lpt_idle.tolist() == widle.tolist()
    exp = port().scale(pred, plen, None, default_profile(), 8, 1, 64, 0.7, 2)
    assert got.n_star == exp["n_star"]
    t = np.array([c.t_total for c in got.candidates])
    assert np.array_equal(bits(t), bits(exp["t_total"]))
