#!/usr/bin/env bash
# The profile captures summarised under profiles/ (run on a B200, e.g.
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/capture_profiles.sh r01c'
# then summarise here with tools/ncu_summary.py). Each ncu pass runs only
# after the same command has exited 0 without ncu.
set -euo pipefail
tag=${1:-rXX}
out=gpurun_out
mkdir -p $out
C="python bench.py --steps 1 --warmup 3 --no-cpu --no-c5"
$C > $out/plain.log 2>&1
# every launch with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file $out/${tag}_launches.csv $C > $out/${tag}_ncu_ll.log 2>&1
python tools/prof_sweep.py 1184 1 > $out/${tag}_sweep_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:lockstep_eval|fast_build|group_table|fast_finish" -c 4 \
    -o $out/${tag}_sweep python tools/prof_sweep.py 1184 1 > $out/${tag}_ncu_sweep.log 2>&1
python tools/prof_dedup.py > $out/${tag}_dedup_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k "regex:compare_stream" -c 1 \
    -o $out/${tag}_dedup python tools/prof_dedup.py > $out/${tag}_ncu_dedup.log 2>&1
# the persistent (cooperative) refinement and the init pass
ncu --set full --clock-control none --import-source on -k "regex:refine_kernel|init_kernel" -c 2 \
    -o $out/${tag}_dedup_refine python tools/prof_dedup.py > $out/${tag}_ncu_dedup_refine.log 2>&1 || true
python tools/prof_trace.py > $out/${tag}_trace_plain.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:classify_kernel|tokens_kernel|nl_write_kernel" -c 3 \
    -o $out/${tag}_trace python tools/prof_trace.py > $out/${tag}_ncu_trace.log 2>&1
