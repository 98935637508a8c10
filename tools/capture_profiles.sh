#!/usr/bin/env bash
# The profile captures summarised under profiles/ (run on a B200, e.g.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/capture_profiles.sh r02b'
# then summarise here with tools/ncu_summary.py and tools/kernel_counters.py).
# Each ncu pass runs only after the same command has exited 0 without ncu.
set -euo pipefail
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
C="python bench.py --steps 1 --warmup 3 --no-cpu --no-c5 --no-c3 --no-arrays --no-check"
$C > $out/${tag}_plain.log 2>&1
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file $out/${tag}_launches.csv $C > $out/${tag}_ncu_ll.log 2>&1
python tools/prof_sweep.py 1184 1 > $out/${tag}_sweep_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:lockstep2|fast_build|group_table|fast_finish" -c 4 \
    -o $out/${tag}_sweep python tools/prof_sweep.py 1184 1 > $out/${tag}_ncu_sweep.log 2>&1
python tools/prof_dedup.py > $out/${tag}_dedup_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:compare_stream|refine_kernel|init_kernel|tables_kernel" -c 4 \
    -o $out/${tag}_dedup python tools/prof_dedup.py > $out/${tag}_ncu_dedup.log 2>&1 || true
python tools/prof_trace.py > $out/${tag}_trace_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:classify_kernel|tokens_kernel|nl_write_kernel" -c 3 \
    -o $out/${tag}_trace python tools/prof_trace.py > $out/${tag}_ncu_trace.log 2>&1
python tools/prof_trace.py jsonl > $out/${tag}_jsonl_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:js_prompt_kernel|js_tokens_kernel|js_depth_kernel|js_child_kernel|js_step" -c 7 \
    -o $out/${tag}_jsonl python tools/prof_trace.py jsonl > $out/${tag}_ncu_jsonl.log 2>&1 || true
