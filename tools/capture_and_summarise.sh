#!/usr/bin/env bash
# capture_profiles.sh, then the text summaries made on the box (the full
# reports together exceed what gpurun brings back): profiles/<tag>_* files
# under gpurun_out/, and the sweep report itself.
set -uo pipefail
tag=${1:-rXX}
out=gpurun_out
bash tools/capture_profiles.sh "$tag"
python tools/ncu_summary.py launches $out/${tag}_launches.csv > $out/${tag}_launches_summary.txt 2>&1
for k in sweep dedup trace jsonl; do
  [ -f $out/${tag}_${k}.ncu-rep ] && python tools/ncu_summary.py report $out/${tag}_${k}.ncu-rep \
      > $out/${tag}_${k}_kernels_full.txt 2>&1
done
cp profiles/kernel_counters.json $out/kernel_counters.prev.json
python tools/kernel_counters.py $out/${tag}_sweep.ncu-rep "$tag" > $out/${tag}_counters.log 2>&1
cp profiles/kernel_counters.json $out/kernel_counters.json
rm -f $out/${tag}_dedup.ncu-rep $out/${tag}_trace.ncu-rep $out/${tag}_jsonl.ncu-rep
ls -la $out
