"""profiles/kernel_counters.json from a committed `ncu --set full` capture of
one sweep batch (tools/prof_sweep.py 1184 1: 1,184 scenarios x 256
candidates), read here with the ncu CLI:

  python tools/kernel_counters.py <sweep.ncu-rep> <tag>

Per kernel: duration, DRAM bytes and warp instructions issued, per launch and
per unit (eval for the evaluator kernels, scenario for the builder). bench.py
multiplies the per-eval figures by its own evals per launch and divides by the
live CUDA-event launch time for the roofline (issue rate, DRAM fraction)."""
import csv
import io
import json
import pathlib
import subprocess
import sys

REPO = pathlib.Path(__file__).resolve().parents[1]
EVALS = 1184 * 256
SCEN = 1184
KEYS = {"dur_ns": "gpu__time_duration.sum", "dram_read": "dram__bytes_read.sum",
        "dram_write": "dram__bytes_write.sum", "inst_issued": "smsp__inst_issued.sum",
        "issue_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
        "cycles": "sm__cycles_elapsed.avg"}
UNIT = {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "cycle": 1, "%": 1}


def main(rep, tag):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    kern = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        name = d["Kernel Name"].split("(")[0].replace("void ", "").split("<")[0].replace("rs::", "")
        rec = {}
        for k, m in KEYS.items():
            v = float(d[m].replace(",", ""))
            rec[k] = v * UNIT.get(u.get(m, ""), 1)
        kern[name] = rec
    ls = kern["lockstep2_kernel"]
    res = {
        "source": f"ncu --set full --clock-control none, tools/prof_sweep.py 1184 1 ({tag}): one "
                  f"launch of each sweep kernel for 1,184 scenarios x 256 candidates",
        "report_summary": f"profiles/{tag}_sweep_kernels_full.txt",
        "evals_per_launch": EVALS,
        "group_eval_inst_issued_per_eval": ls["inst_issued"] / EVALS,
        "group_eval_dram_bytes_per_eval": (ls["dram_read"] + ls["dram_write"]) / EVALS,
        "group_eval_issue_pct_active": ls["issue_pct"],
        "kernels": kern,
    }
    fb = kern.get("fast_build_kernel")
    if fb:
        res["fast_build_dram_bytes_per_scenario"] = (fb["dram_read"] + fb["dram_write"]) / SCEN
        res["fast_build_inst_issued_per_scenario"] = fb["inst_issued"] / SCEN
    old = REPO / "profiles" / "kernel_counters.json"
    if old.exists():  # keep the dedup / trace figures of earlier captures
        prev = json.loads(old.read_text())
        for k, v in prev.items():
            if k.startswith(("dedup_", "trace_")):
                res.setdefault(k, v)
    old.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps({k: v for k, v in res.items() if k != "kernels"}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "rXX")
