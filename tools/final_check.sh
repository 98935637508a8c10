#!/usr/bin/env bash
# GPU suite, smoke() and the default bench line of the current build, with
# the headline fields echoed (run on a B200 box: gpurun -- bash tools/final_check.sh TAG)
set -uo pipefail
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
python -m pytest tests -m gpu -q > $out/gpu_tests_${tag}.log 2>&1
tail -2 $out/gpu_tests_${tag}.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py > $out/bench_${tag}_n1.json 2> $out/bench_${tag}_n1.err
python - "$out/bench_${tag}_n1.json" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
print({"value": d["value"], "e2e": d["e2e"]["value"], "frac": d["roofline"]["frac"],
       "parity": d["parity_sampled"], "c5": d["c5"]["value"], "trace": d["trace"]["value"],
       "jsonl": d["trace"]["jsonl"]["value"], "trace_parity": [d["trace"].get("parity"), d["trace"]["jsonl"].get("parity")],
       "clocks": d["clocks"]})
PY
