#!/usr/bin/env bash
# Reference vs patched simulator on C5 steps in all three cut modes (CPU only;
# needs /root/reference, oracle/_ref and build/shim/simulator_b200.cpp from
# `make -C oracle ref` and `make shim`): bash tools/sim_compare.sh [steps=12]
set -euo pipefail
steps=${1:-12}
R=/root/reference/proj
O=oracle/_ref/obj
out=build/sim_compare
mkdir -p $out
INC="-I$R/include -Ioracle/include_shim -I/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
CX="g++ -std=c++20 -O2 -DNDEBUG $INC"
objs="$O/workload.o $O/predictor.o $O/dedup.o $O/profile.o $O/planner.o $O/placement.o $O/training.o $O/report.o $O/cli.o"
$CX -c build/shim/simulator_b200.cpp -o $out/sim_b200.o
$CX tools/sim_compare.cpp $objs $O/simulator.o -o $out/cmp_ref -lpthread
$CX tools/sim_compare.cpp $objs $out/sim_b200.o -o $out/cmp_b200 -lpthread
$out/cmp_ref "$steps" > $out/ref.txt &
$out/cmp_b200 "$steps" > $out/b200.txt
wait
wc -l $out/ref.txt
cmp $out/ref.txt $out/b200.txt && echo "identical: events, segments, releases ($steps steps x 3 cut modes)"
