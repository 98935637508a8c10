"""CPU suite: pin the C restatement (oracle/rs_oracle.c) against the
reference itself (oracle/_ref, when it was built here) and against the
committed golden vectors (tests/golden/, made by tests/golden/make_golden.py
from the reference). No GPU needed."""
import json
import pathlib

import numpy as np
import pytest

from cases import (Rng, c4_spec, constant_profile, csr, profiles, random_batch,
                   random_predicted, small_profile)
from oracle_lib import OracleError, port, ref
from paper_2602_22718_b200.rollsim import default_profile

GOLDEN = pathlib.Path(__file__).parent / "golden"


def bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, np.float64)]


needs_ref = pytest.mark.skipif(ref() is None, reason="reference not built (no /root/reference)")


# ------------------------------------------------------------ golden pins
def load(name):
    return json.loads((GOLDEN / name).read_text())


def test_golden_tpot():
    g = load("tpot.json")
    for name, prof in profiles().items():
        case = g[name]
        out = port().tpot_seconds(prof, case["b"], case["c"])
        assert hexs(out) == case["tpot"], name


def test_golden_prefix():
    for case in load("prefix.json"):
        tok, off = np.array(case["tok"], np.int32), np.array(case["off"], np.int64)
        info, u, t, r = port().prefix_curves(tok, off, case["n_l"])
        assert info.tolist() == case["info"]
        assert u.tolist() == case["ucount"] and t.tolist() == case["utokens"] and r.tolist() == case["rem"]
        assert list(port().select_prefix_length(tok, off, case["cap"], 1, case["info"][2])) == case["select"]
        raw, dd, fr = port().dedup_savings(tok, off, case["l_star"], case["g"])
        assert [raw, dd, float(fr).hex()] == case["savings"]
        assert port().unique_prefix_count_among(tok, off, case["among_l"]) == case["among"]


def test_golden_planner():
    for case in load("planner.json"):
        prof = profiles()[case["profile"]]
        pred, plen = np.array(case["pred"]), np.array(case["plen"], np.int32)
        out = port().scale(pred, plen, None, prof, case["g"], case["n_min"], case["n_max"],
                           case["lambda"], case["gpus"])
        assert out["n_star"] == case["n_star"]
        assert hexs(out["t_total"]) == case["t_total"]
        assert hexs(out["cost"]) == case["cost"]
        assert hexs(out["score"]) == case["score"]
        assert out["order"].tolist() == case["order"]
        assert port().integrate(plen, pred, prof).hex() == case["integrate"]


def test_golden_c4_scenario():
    """A C4 scenario (4096 prompts) scaled by the reference over N in [1, 64]."""
    g = load("c4_scenario.json")
    pred, plen = port().generate_scenarios(c4_spec(1, count=g["count"], first=g["scenario"]))
    assert hex(int(bits(pred).sum() & np.uint64(2**64 - 1))) == g["pred_checksum"]
    assert int(plen.astype(np.int64).sum()) == g["plen_sum"]
    out = port().scale(pred, plen, None, default_profile(), 8, 1, g["n_max"], 0.7, 2)
    assert out["n_star"] == g["n_star"]
    assert hexs(out["t_total"]) == g["t_total"]
    assert hexs(out["cost"]) == g["cost"]


# --------------------------------------------- known answers from the reference tests
def test_known_answers_dedup():
    o = port()
    tok, off = csr([[1, 2, 3], [1, 2, 4], [7, 8, 9]])  # test_dedup.cpp:78-94
    info, u, _, _ = o.prefix_curves(tok, off, 10)
    assert u[:3].tolist() == [2, 2, 3] and u[9] == 3 and info.tolist() == [3, 3, 3, 9]
    tok, off = csr([[1, 1, 1], [1, 1, 2], [1, 2, 3], [1, 2, 4]])  # :150-185
    assert o.select_prefix_length(tok, off, 2, 1, 3) == (2, False)
    assert o.select_prefix_length(tok, off, 4, 1, 3) == (3, False)
    with pytest.raises(OracleError) as e:
        o.select_prefix_length(tok, off, 0, 1, 3)
    assert e.value.status == 2
    tok, off = csr([[1, 2, 3, 4]] * 3)  # :220-233 and acceptance crit. 1
    assert o.dedup_savings(tok, off, 4, 1)[:2] == (12, 4)
    tok, off = csr([[1, 2], [1, 2, 3]])  # :260-274
    raw, dd, fr = o.dedup_savings(tok, off, 2, 1)
    assert (raw, dd) == (5, 3) and abs(fr - 0.4) < 1e-15
    seqs = [[i * 100 + k for k in range(5 + i)] for i in range(6)]  # acceptance_main.cpp:54-74
    tok, off = csr(seqs)
    raw, dd, fr = o.dedup_savings(tok, off, 10, 3)
    assert fr == 2.0 / 3.0


def test_known_answers_planner():
    o = port()
    flat = constant_profile(0.01)
    assert abs(o.integrate([10], [100.0], flat) - 1.0) < 1e-12  # test_planner.cpp:115-124
    assert abs(o.integrate([10, 10], [100.0, 50.0], flat) - 1.0) < 1e-12
    assert abs(o.integrate([10], [99.2], flat) - 1.0) < 1e-12
    assert o.integrate([], [], flat) == 0.0
    with pytest.raises(OracleError):
        o.integrate([10], [0.0], flat)
    order, goff = o.assign([100, 90, 10, 5], None, 2)  # :61-77
    assert order.tolist() == [0, 1, 2, 3] and goff.tolist() == [0, 2, 4]
    order, goff = o.assign([50, 50, 50, 50], [3, 1, 0, 2], 2)  # ties by id: a, m | q, z
    assert order.tolist() == [2, 1, 3, 0]
    order, goff = o.assign([100 - i for i in range(7)], None, 3)  # :93-106
    assert goff.tolist() == [0, 3, 5, 7]
    cost, _ = o.estimate_cost([10], [100.0], [0, 1], [2], constant_profile(0.1, 0.1, 2), 1)
    assert abs(cost - 2.0) < 1e-12  # :186-196
    for args in [(0, 2, 0.5), (2, 1, 0.5), (1, 3, 0.5)]:  # :334-342
        with pytest.raises(OracleError) as e:
            o.scale([10, 20], [10, 10], None, flat, 1, args[0], args[1], args[2], 2)
        assert e.value.status == 1
    for lam in (-0.1, 1.1):
        with pytest.raises(OracleError) as e:
            o.scale([10, 20], [10, 10], None, flat, 1, 1, 2, lam, 2)
        assert e.value.status == 2
    r = o.scale([100.0] * 8, [10] * 8, None, flat, 1, 2, 4, 0.7, 2)  # :249-261
    assert r["n_star"] == 2 and np.all(r["t_norm"] == 0.0)


# ----------------------------------------------- port == reference, bitwise
@needs_ref
def test_port_matches_reference_tpot():
    rng = Rng(11)
    for name, prof in profiles().items():
        b = [rng.uniform_range(0.1, 600.0) for _ in range(500)] + list(range(1, 300))
        c = [rng.uniform_range(0.0, 8000.0) for _ in range(500)] + list(range(0, 5980, 20))
        assert np.array_equal(bits(port().tpot_seconds(prof, b, c)),
                              bits(ref().tpot_seconds(prof, b, c))), name


@needs_ref
def test_port_matches_reference_prefix_random():
    rng = Rng(2026)
    for trial in range(120):
        seqs = random_batch(rng, max_count=20, max_len=12, alphabet=3)
        tok, off = csr(seqs)
        a = port().prefix_curves(tok, off, 14)
        b = ref().prefix_curves(tok, off, 14)
        for x, y in zip(a, b):
            assert x.tolist() == y.tolist(), trial
        cap = rng.uniform_int(1, 8)
        assert port().select_prefix_length(tok, off, cap, 1, int(a[0][2])) == \
            ref().select_prefix_length(tok, off, cap, 1, int(a[0][2]))
        l = rng.uniform_int(1, 13)
        assert port().dedup_savings(tok, off, l, 3) == ref().dedup_savings(tok, off, l, 3)
        assert port().unique_prefix_count_among(tok, off, l) == ref().unique_prefix_count_among(tok, off, l)


@needs_ref
def test_port_matches_reference_planner_random():
    rng = Rng(88)
    for trial in range(60):
        count = rng.uniform_int(2, 40)
        pred, plen = random_predicted(rng, count, 1.0, 900.0, 1, 900, integer=trial % 3 == 0)
        rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
        prof = [default_profile(), small_profile(), constant_profile(0.01)][trial % 3]
        n_max = rng.uniform_int(1, count)
        lam = [0.0, 0.25, 0.7, 1.0][trial % 4]
        g = rng.uniform_int(1, 8)
        a = port().scale(pred, plen, rank, prof, g, 1, n_max, lam, 2)
        b = ref().scale(pred, plen, rank, prof, g, 1, n_max, lam, 2)
        assert a["n_star"] == b["n_star"], trial
        for k in ("t_total", "cost", "t_norm", "c_norm", "score"):
            assert np.array_equal(bits(a[k]), bits(b[k])), (trial, k)
        assert a["order"].tolist() == b["order"].tolist()
        assert np.array_equal(bits(a["actor_times"]), bits(b["actor_times"]))
        assert port().integrate(plen, pred, prof) == ref().integrate(plen, pred, prof)
        assert port().estimate_actor_time(plen, pred, prof, g) == ref().estimate_actor_time(plen, pred, prof, g)
        o1, g1 = port().assign(pred, rank, n_max)
        o2, g2 = ref().assign(pred, rank, n_max)
        assert o1.tolist() == o2.tolist() and g1.tolist() == g2.tolist()


@needs_ref
def test_port_matches_reference_c3_sized():
    """One C4 scenario at 4096 prompts, N in [1, 128], bitwise."""
    pred, plen = port().generate_scenarios(c4_spec(1, count=4096, first=7))
    a = port().scale(pred, plen, None, default_profile(), 8, 1, 128, 0.7, 2)
    b = ref().scale(pred, plen, None, default_profile(), 8, 1, 128, 0.7, 2)
    assert a["n_star"] == b["n_star"]
    assert np.array_equal(bits(a["t_total"]), bits(b["t_total"]))
    assert np.array_equal(bits(a["cost"]), bits(b["cost"]))


@needs_ref
def test_port_matches_reference_placement_penalty():
    """scale() with plan_rlhfless's placement penalty: the C restatement
    against the reference's own place() / check_overlap(), bitwise."""
    from cases import placement_cases
    rng = Rng(515)
    for ci, (pen, gpus, cap) in enumerate(placement_cases()):
        for trial in range(6):
            count = rng.uniform_int(cap, 60)
            pred, plen = random_predicted(rng, count, 1.0, 900.0, 1, 900, integer=trial % 2 == 0)
            rank = np.random.RandomState(trial).permutation(count).astype(np.int32)
            prof = [default_profile(), small_profile()][trial % 2]
            n_max = min(cap, count)
            a = port().scale_placed(pred, plen, rank, prof, 4, 1, n_max, 0.6, gpus, pen)
            b = ref().scale_placed(pred, plen, rank, prof, 4, 1, n_max, 0.6, gpus, pen)
            assert a["n_star"] == b["n_star"], (ci, trial)
            for k in ("t_total", "t_penalty", "cost", "t_norm", "c_norm", "score"):
                assert np.array_equal(bits(a[k]), bits(b[k])), (ci, trial, k)
            assert a["order"].tolist() == b["order"].tolist()


@needs_ref
def test_placement_penalty_errors_match_reference():
    from cases import placement_cases
    from paper_2602_22718_b200.rollsim import ClusterTopology, PlacementPenalty
    pen, gpus, cap = placement_cases()[0]
    pred, plen = random_predicted(Rng(3), 40)
    for o in (port(), ref()):
        with pytest.raises(OracleError) as e:  # more actors than the cluster hosts
            o.scale_placed(pred, plen, None, default_profile(), 2, 1, cap + 1, 0.5, gpus, pen)
        assert e.value.status == 6
        bad = PlacementPenalty(ClusterTopology([8, 8], intra_node_bw=1e9, inter_node_bw=2e9),
                               l_prefill_seconds=0.1)
        with pytest.raises(OracleError) as e:
            o.scale_placed(pred, plen, None, default_profile(), 2, 1, 4, 0.5, gpus, bad)
        assert e.value.status == 2
        with pytest.raises(OracleError) as e:  # scale's own checks come first
            o.scale_placed(pred, plen, None, default_profile(), 2, 1, 41, 0.5, gpus, bad)
        assert e.value.status == 1


@needs_ref
def test_port_matches_reference_predictor():
    """The C restatement of LengthHistory::predict / predict_noisy against
    the reference's own LengthHistory (loaded via from_json), bitwise."""
    from cases import predictor_cases
    for t, (w, a, m, obs, depth, gt, ids, noise) in enumerate(predictor_cases()):
        x = port().predict_lengths(obs, depth, gt, w, a, m, noise, ids)
        y = ref().predict_lengths(obs, depth, gt, w, a, m, noise, ids)
        assert np.array_equal(bits(x), bits(y)), t
        if noise is not None and noise.bucket_accuracy == 0.0 and m > noise.bucket_width:
            assert (x != port().predict_lengths(obs, depth, gt, w, a, m)).any(), t


@needs_ref
def test_predictor_config_errors_match_reference():
    from paper_2602_22718_b200.rollsim import NoiseModel
    obs, depth, gt = np.zeros((1, 1)), np.zeros(1, np.int32), np.ones(1, np.int32)
    for o in (port(), ref()):
        for args in ((0, 0.5, 10, None), (1, 0.0, 10, None), (1, 0.5, 0, None),
                     (1, 0.5, 10, NoiseModel("bucket", 1.5, 5, 0)),
                     (1, 0.5, 10, NoiseModel("bucket", 0.5, 11, 0))):
            with pytest.raises(OracleError) as e:
                o.predict_lengths(obs, depth, gt, *args[:3], args[3], ["p0"])
            assert e.value.status == 2, args


@needs_ref
def test_reference_trace_reader_wrapper():
    """The trace oracle (ref_trace_prompts) returns the reference reader's
    id-sorted prompt table, limits and error types."""
    from cases import trace_csv
    text = trace_csv([("b", 5, [1, 2, 3]), ("a", 9, ["4", "7x"])], g=3, max_prompt_len=8)
    t = ref().trace_prompts(text)
    assert t["ids"] == ["a", "b"] and t["gt"].tolist() == [9, 5]
    assert t["offsets"].tolist() == [0, 2, 5] and t["tokens"].tolist() == [4, 7, 1, 2, 3]
    assert (t["g"], t["max_prompt_len"], t["max_response_len"]) == (3, 8, 2048)
    with pytest.raises(OracleError) as e:
        ref().trace_prompts(trace_csv([("a", 1, [1])], header=False))
    assert e.value.status == 7


@needs_ref
def test_reference_trace_steps_and_jsonl_wrappers():
    """ref_trace_steps lays the step table out as rs_trace_csr_steps_copy
    does (batch order, indices into the id-sorted table, g lengths per
    entry), for both formats; ref_trace_convert round-trips CSV <-> JSONL."""
    from cases import trace_csv
    text = trace_csv([("b", 5, [1, 2, 3]), ("a", 9, [4])], g=2,
                     steps=[(0, [("b", [7, 8]), ("a", [5, 6])]), (3, [("a", [1, 2])])])
    s = ref().trace_steps(text)
    assert s["step_idx"].tolist() == [0, 3] and s["entry_off"].tolist() == [0, 2, 3]
    assert s["entry_prompt"].tolist() == [1, 0, 0]
    assert s["lengths"].tolist() == [[7, 8], [5, 6], [1, 2]]
    jsonl = ref().trace_convert(text, "csv", "jsonl")
    assert jsonl.startswith(b'{"g":2') and b'"type":"header"' in jsonl
    j = ref().trace_steps(jsonl, "jsonl")
    # JSONL keeps the batch order in "scheduled" next to the id-keyed lengths
    assert j["step_idx"].tolist() == [0, 3] and j["entry_prompt"].tolist() == [1, 0, 0]
    assert j["lengths"].tolist() == [[7, 8], [5, 6], [1, 2]]
    assert ref().trace_convert(jsonl, "jsonl", "csv") == ref().trace_convert(text, "csv", "csv")
    with pytest.raises(OracleError) as e:
        ref().trace_steps(b'{"type":"header","g":1,"prompts":[]}\n{"step":0}\n', "jsonl")
    assert e.value.status == 7
