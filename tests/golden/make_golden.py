"""Regenerate the golden vectors in tests/golden/ FROM THE REFERENCE ITSELF.

Runs the unmodified reference library (oracle/_ref/librollsim_ref_capi.so,
built by `make -C oracle ref` from /root/reference/proj/src) on seeded
inputs and writes small JSON fixtures. Floating-point values are stored as
exact hex strings. Usage: python tests/golden/make_golden.py
"""
import json
import pathlib
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

from cases import Rng, c4_spec, csr, profiles, random_batch, random_predicted  # noqa: E402
from oracle_lib import port, ref  # noqa: E402
from paper_2602_22718_b200.rollsim import default_profile  # noqa: E402


def hexs(a):
    return [float(x).hex() for x in np.asarray(a, np.float64)]


def main():
    R = ref()
    assert R is not None, "reference not built"
    # tpot at integer and fractional points for the three test profiles
    rng = Rng(5)
    tp = {}
    for name, prof in profiles().items():
        b = [float(x) for x in (0.5, 1, 2, 3, 7, 8, 100, 256, 300, 1000)] + \
            [rng.uniform_range(0.1, 500.0) for _ in range(40)]
        c = [float(x) for x in (1, 10, 127, 128, 300, 511, 512, 1024, 4096, 99999)] + \
            [rng.uniform_range(0.0, 6000.0) for _ in range(40)]
        tp[name] = {"b": b, "c": c, "tpot": hexs(R.tpot_seconds(prof, b, c))}
    (HERE / "tpot.json").write_text(json.dumps(tp))

    # dedup: random ragged batches over a small alphabet (test_dedup.cpp:52-65)
    rng = Rng(31337)
    cases = []
    for trial in range(40):
        seqs = random_batch(rng, max_count=20, max_len=12, alphabet=3)
        tok, off = csr(seqs)
        info, u, t, r = R.prefix_curves(tok, off, 14)
        cap = rng.uniform_int(1, 8)
        l_star = rng.uniform_int(1, 13)
        g = rng.uniform_int(1, 4)
        among_l = rng.uniform_int(1, 13)
        raw, dd, fr = R.dedup_savings(tok, off, l_star, g)
        cases.append({"tok": tok.tolist(), "off": off.tolist(), "n_l": 14, "info": info.tolist(),
                      "ucount": u.tolist(), "utokens": t.tolist(), "rem": r.tolist(), "cap": cap,
                      "select": list(R.select_prefix_length(tok, off, cap, 1, int(info[2]))),
                      "l_star": l_star, "g": g, "savings": [raw, dd, float(fr).hex()],
                      "among_l": among_l, "among": R.unique_prefix_count_among(tok, off, among_l)})
    (HERE / "prefix.json").write_text(json.dumps(cases))

    # planner: random scale instances on the three profiles
    rng = Rng(4242)
    cases = []
    for trial in range(30):
        name = ["default", "small", "constant"][trial % 3]
        prof = profiles()[name]
        count = rng.uniform_int(2, 24)
        pred, plen = random_predicted(rng, count, 1.0, 700.0, 1, 900, integer=trial % 4 == 0)
        n_max = rng.uniform_int(1, count)
        lam = [0.0, 0.3, 0.7, 1.0][trial % 4]
        g = rng.uniform_int(1, 8)
        out = R.scale(pred, plen, None, prof, g, 1, n_max, lam, 2)
        cases.append({"profile": name, "pred": [float(x) for x in pred], "plen": plen.tolist(),
                      "g": g, "n_min": 1, "n_max": n_max, "lambda": lam, "gpus": 2,
                      "n_star": out["n_star"], "t_total": hexs(out["t_total"]),
                      "cost": hexs(out["cost"]), "score": hexs(out["score"]),
                      "order": out["order"].tolist(),
                      "integrate": R.integrate(plen, pred, prof).hex()})
    (HERE / "planner.json").write_text(json.dumps(cases))

    # one C4 scenario (scenario generator = DESIGN.md §4.1), 4096 prompts
    count, scen, n_max = 4096, 3, 64
    pred, plen = port().generate_scenarios(c4_spec(1, count=count, first=scen))
    out = R.scale(pred, plen, None, default_profile(), 8, 1, n_max, 0.7, 2)
    bsum = int(pred.view(np.uint64).sum() & np.uint64(2**64 - 1))
    (HERE / "c4_scenario.json").write_text(json.dumps({
        "count": count, "scenario": scen, "n_max": n_max, "pred_checksum": hex(bsum),
        "plen_sum": int(plen.astype(np.int64).sum()), "n_star": out["n_star"],
        "t_total": hexs(out["t_total"]), "cost": hexs(out["cost"])}))
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
