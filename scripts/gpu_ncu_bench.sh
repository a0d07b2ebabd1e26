#!/bin/bash
# One ncu --set full capture of the dominant kernel + the default bench line.
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s 2 -c 1 \
  -o gpurun_out/ncu_C2_${TAG} -f python scripts/profile_run.py C2 2048 > gpurun_out/ncu_C2_${TAG}.log 2>&1
echo "ncu exit $?"
if [ "${2:-}" != "nobench" ]; then timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?"; cat gpurun_out/bench.log; fi
