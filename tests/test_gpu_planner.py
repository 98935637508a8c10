"""GPU parity: assignment (2) and actor scaling (3) through the C-ABI,
bit-exact against the CPU oracle (oracle/rs_oracle.c, itself pinned to the
reference in tests/test_oracle.py) on the same seeded inputs."""
import numpy as np
import pytest

import paper_2602_22718_b200.rollsim as rs
from cases import Rng, c4_spec, constant_profile, profiles, random_predicted, small_profile
from oracle_lib import port, ref
from paper_2602_22718_b200.rollsim import (ActorGroup, PredictedPrompt, ResponseSpec,
                                           default_profile)

pytestmark = pytest.mark.gpu


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


def pp(i, pred, plen=10):
    return PredictedPrompt(f"p{i:06d}", plen, pred)


# --------------------------------------------------------------- tpot
@pytest.mark.parametrize("name", ["default", "small", "constant"])
def test_tpot_bitwise(name):
    prof = profiles()[name]
    rng = Rng(3)
    b = [rng.uniform_range(0.1, 600.0) for _ in range(2000)] + [float(x) for x in range(0, 400)]
    c = [rng.uniform_range(0.0, 9000.0) for _ in range(2000)] + [float(x) for x in range(0, 8000, 20)]
    assert same(prof.tpot_seconds(b, c), port().tpot_seconds(prof, b, c))


# ------------------------------------------------------- reference known answers
def test_assign_golden_splits():
    """proj/tests/test_planner.cpp:61-106."""
    ps = [PredictedPrompt("a", 10, 100), PredictedPrompt("b", 10, 90),
          PredictedPrompt("c", 10, 10), PredictedPrompt("d", 10, 5)]
    g = rs.assign(ps, 2, 2)
    assert [x.prompt_ids for x in g] == [["a", "b"], ["c", "d"]]
    assert g[0].predicted_lengths == [100, 90] and g[0].gpu_count == 2
    one = rs.assign(ps, 1, 4)
    assert one[0].prompt_ids == ["a", "b", "c", "d"] and one[0].gpu_count == 4
    shuffled = [ps[3], ps[1], ps[0], ps[2]]
    assert [x.prompt_ids for x in rs.assign(shuffled, 2, 2)] == [["a", "b"], ["c", "d"]]
    tied = [PredictedPrompt(i, 10, 50) for i in "zmaq"]
    assert [x.prompt_ids for x in rs.assign(tied, 2, 2)] == [["a", "m"], ["q", "z"]]
    seven = [PredictedPrompt(f"p{i}", 10, 100 - i) for i in range(7)]
    g = rs.assign(seven, 3, 2)
    assert [x.prompt_ids for x in g] == [["p0", "p1", "p2"], ["p3", "p4"], ["p5", "p6"]]
    with pytest.raises(rs.ValidationError):
        rs.assign([], 1, 2)
    with pytest.raises(rs.ValidationError):
        rs.assign([ps[0]], 0, 2)
    with pytest.raises(rs.ValidationError):
        rs.assign([ps[0]], 2, 2)


def test_integrate_known_answers():
    """proj/tests/test_planner.cpp:115-133."""
    flat = constant_profile(0.01)
    assert rs.integrate_decode_seconds([ResponseSpec(10, 100.0)], flat) == pytest.approx(1.0)
    assert rs.integrate_decode_seconds([ResponseSpec(10, 100.0), ResponseSpec(10, 50.0)],
                                       flat) == pytest.approx(1.0)
    assert rs.integrate_decode_seconds([ResponseSpec(10, 99.2)], flat) == pytest.approx(1.0)
    with pytest.raises(rs.ValidationError):
        rs.integrate_decode_seconds([ResponseSpec(10, 0.0)], flat)
    assert rs.integrate_decode_seconds([], flat) == 0.0


def naive_decode_seconds(responses, prof):
    """Tick-by-tick reference (proj/tests/test_planner.cpp:37-57)."""
    last = max(int(np.ceil(r.target_len)) for r in responses)
    b = []
    c = []
    for t in range(1, last + 1):
        live = [r for r in responses if int(np.ceil(r.target_len)) >= t]
        b.append(float(len(live)))
        c.append(max(float(r.prompt_len) + float(t - 1) for r in live))
    return float(np.sum(port().tpot_seconds(prof, b, c)))


def test_integrate_matches_tick_by_tick():
    """proj/tests/test_planner.cpp:135-152 (1e-9)."""
    prof = default_profile()
    rng = Rng(404)
    for trial in range(50):
        rs_ = [ResponseSpec(rng.uniform_int(1, 900), rng.uniform_range(1.0, 600.0))
               for _ in range(rng.uniform_int(1, 12))]
        fast = rs.integrate_decode_seconds(rs_, prof)
        assert fast == pytest.approx(naive_decode_seconds(rs_, prof), rel=1e-9), trial


def test_actor_time_and_cost():
    """proj/tests/test_planner.cpp:154-208."""
    flat = constant_profile(0.01)
    g = ActorGroup(0, ["a", "b"], [10, 10], [100.0, 50.0], 2)
    assert rs.estimate_actor_time(g, flat, 1) == pytest.approx(1.0)
    assert rs.estimate_actor_time(g, flat, 4) == pytest.approx(1.0)
    with pytest.raises(rs.ValidationError):
        rs.estimate_actor_time(g, flat, 0)
    prof = default_profile()
    assert rs.estimate_actor_time(g, prof, 4) > rs.estimate_actor_time(g, prof, 1)
    g3 = ActorGroup(0, ["a", "b", "c"], [300, 100, 50], [400.0, 250.0, 30.0], 1)
    rev = ActorGroup(0, g3.prompt_ids[::-1], g3.prompt_lens[::-1], g3.predicted_lengths[::-1], 1)
    assert rs.estimate_actor_time(g3, prof, 2) == rs.estimate_actor_time(rev, prof, 2)
    fl = constant_profile(0.1, 0.1, 2)
    one = ActorGroup(0, ["a"], [10], [100.0], 2)
    assert rs.estimate_cost([one], fl, 1) == pytest.approx(2.0, rel=1e-12)
    two = ActorGroup(1, ["a"], [10], [50.0], 2)
    assert rs.estimate_cost([one, two], fl, 1) == pytest.approx(
        rs.estimate_cost([one], fl, 1) + rs.estimate_cost([two], fl, 1), rel=1e-12)


def test_scale_degenerate_and_validation():
    """proj/tests/test_planner.cpp:249-273, 334-342."""
    flat = constant_profile(0.01)
    ps = [pp(i, 100.0) for i in range(8)]
    r = rs.scale(ps, flat, 1, 2, 4, 0.7, 2)
    assert r.n_star == 2 and all(c.t_norm == 0.0 for c in r.candidates)
    tied = rs.scale(ps, flat, 1, 2, 4, 1.0, 2)
    assert tied.n_star == 2 and all(c.score == 0.0 for c in tied.candidates)
    single = rs.scale(ps, flat, 1, 3, 3, 0.5, 2)
    assert single.n_star == 3 and len(single.candidates) == 1
    two = [pp(0, 10), pp(1, 20)]
    for a, b, lam in [(0, 2, 0.5), (2, 1, 0.5), (1, 3, 0.5)]:
        with pytest.raises(rs.ValidationError):
            rs.scale(two, flat, 1, a, b, lam, 2)
    for lam in (-0.1, 1.1):
        with pytest.raises(rs.ConfigError):
            rs.scale(two, flat, 1, 1, 2, lam, 2)
    with pytest.raises(rs.ValidationError):
        rs.scale([pp(0, 0.5), pp(1, 3.0)], flat, 1, 1, 2, 0.5, 2)


def test_scale_penalty_steers():
    """proj/tests/test_planner.cpp:358-376."""
    prof = default_profile()
    ps = [pp(i, 40.0 + 35.0 * i, 150) for i in range(12)]
    plain = rs.scale(ps, prof, 2, 1, 6, 1.0, 2)
    assert plain.n_star > 1
    seen = []

    def veto(n, groups, times):
        seen.append((n, len(groups), len(times)))
        return 1e6 if n > 1 else 0.0

    steered = rs.scale(ps, prof, 2, 1, 6, 1.0, 2, veto)
    assert steered.n_star == 1
    assert seen == [(n, n, n) for n in range(1, 7)]
    for c in steered.candidates:
        if c.n_actors > 1:
            assert c.t_penalty == pytest.approx(1e6)


# ------------------------------------------------ bitwise vs the oracle
def check_scale(pred, plen, rank, prof, g, n_min, n_max, lam, gpus=2, penalty=None):
    ids = [f"r{int(x):010d}" for x in (rank if rank is not None else range(len(pred)))]
    ps = [PredictedPrompt(ids[i], int(plen[i]), float(pred[i])) for i in range(len(pred))]
    got = rs.scale(ps, prof, g, n_min, n_max, lam, gpus)
    want = port().scale(pred, plen, rank, prof, g, n_min, n_max, lam, gpus)
    assert got.n_star == want["n_star"]
    for k in ("t_total", "cost", "t_norm", "c_norm", "score"):
        assert same([getattr(c, k) for c in got.candidates], want[k]), k
    assert same(got.actor_times, want["actor_times"])
    order = [int(ids.index(i)) for grp in got.groups for i in grp.prompt_ids]
    assert order == want["order"].tolist()
    return got


def test_scale_random_bitwise():
    rng = Rng(88)
    for trial in range(40):
        count = rng.uniform_int(2, 60)
        pred, plen = random_predicted(rng, count, 1.0, 900.0, 1, 900, integer=trial % 3 == 0)
        rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
        prof = [default_profile(), small_profile(), constant_profile(0.01)][trial % 3]
        n_max = rng.uniform_int(1, count)
        n_min = rng.uniform_int(1, n_max)
        check_scale(pred, plen, rank, prof, rng.uniform_int(1, 8), n_min, n_max,
                    [0.0, 0.25, 0.7, 1.0][trial % 4])


def test_scale_unbounded_predictions_use_generic_path():
    """Predictions above the bucketed range (> 16384 ticks) and exact ties."""
    rng = Rng(9)
    pred, plen = random_predicted(rng, 300, 1.0, 60000.0, 1, 2000)
    pred[::7] = 5000.0  # ties broken by id
    check_scale(pred, plen, np.random.RandomState(1).permutation(300).astype(np.int32),
                default_profile(), 8, 1, 40, 0.7)


def test_integrate_and_cost_random_bitwise():
    rng = Rng(77)
    for trial in range(30):
        n = rng.uniform_int(1, 200)
        pred, plen = random_predicted(rng, n, 1.0, 3000.0, 0, 1500, integer=trial % 2 == 0)
        prof = [default_profile(), small_profile(), constant_profile(0.02)][trial % 3]
        got = rs.integrate_decode_seconds([ResponseSpec(int(a), float(b)) for a, b in zip(plen, pred)], prof)
        assert same([got], [port().integrate(plen, pred, prof)])
        g = rng.uniform_int(1, 8)
        grp = ActorGroup(0, [str(i) for i in range(n)], plen.tolist(), pred.tolist(), 2)
        assert same([rs.estimate_actor_time(grp, prof, g)], [port().estimate_actor_time(plen, pred, prof, g)])
        cuts = sorted({0, n, *[rng.uniform_int(0, n) for _ in range(3)]})
        groups = [ActorGroup(k, [str(i) for i in range(a, b)], plen[a:b].tolist(), pred[a:b].tolist(), k + 1)
                  for k, (a, b) in enumerate(zip(cuts[:-1], cuts[1:]))]
        times = []
        cost = rs.estimate_cost(groups, prof, g, times)
        wc, wt = port().estimate_cost(plen, pred, cuts, [k + 1 for k in range(len(groups))], prof, g)
        assert same([cost], [wc]) and same(times, wt)


def test_assign_random_matches_oracle():
    rng = Rng(5)
    for trial in range(20):
        count = rng.uniform_int(1, 5000)
        pred, _ = random_predicted(rng, count, -50.0, 20000.0, integer=trial % 2 == 0)
        rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
        n = rng.uniform_int(1, count)
        ids = [f"r{int(x):010d}" for x in rank]
        groups = rs.assign([PredictedPrompt(ids[i], 0, float(pred[i])) for i in range(count)], n, 2)
        want_order, want_off = port().assign(pred, rank, n)
        got = [ids.index(i) for grp in groups for i in grp.prompt_ids] if count < 400 else None
        if got is not None:
            assert got == want_order.tolist()
        assert [len(g.prompt_ids) for g in groups] == np.diff(want_off).tolist()


@pytest.mark.slow
def test_scale_c3_full_size_bitwise():
    """C3: 64K prompts x G=8 onto N in [1, 512], bitwise vs the oracle."""
    pred, plen = port().generate_scenarios(c4_spec(1, count=65536, first=0))
    got = check_scale(pred, plen, None, default_profile(), 8, 1, 512, 0.7)
    idle = port().scale_idle(pred, None, 8, 1, 512)
    assert np.array_equal(got.idle_slot_ticks, idle)


def test_scale_against_reference_when_available():
    R = ref()
    if R is None:
        pytest.skip("reference library not shipped to this box")
    pred, plen = port().generate_scenarios(c4_spec(1, count=4096, first=11))
    got = rs.scale([PredictedPrompt(f"p{i:06d}", int(plen[i]), float(pred[i])) for i in range(4096)],
                   default_profile(), 8, 1, 96, 0.7, 2)
    want = R.scale(pred, plen, None, default_profile(), 8, 1, 96, 0.7, 2)
    assert got.n_star == want["n_star"]
    assert same([c.t_total for c in got.candidates], want["t_total"])
    assert same([c.cost for c in got.candidates], want["cost"])


def test_lpt_matches_oracle():
    rng = Rng(12)
    for trial in range(6):
        count = rng.uniform_int(1, 3000)
        pred, _ = random_predicted(rng, count, 1.0, 16000.0, integer=trial % 2 == 0)
        rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
        g = rng.uniform_int(1, 8)
        n_max = [7, 40, 100, 300, 700, 1024][trial]
        mk, idle = rs.lpt(pred, rank, g, 1, n_max)
        wmk, widle = port().lpt(pred, rank, g, 1, n_max)
        assert mk.tolist() == wmk.tolist() and idle.tolist() == widle.tolist(), trial
