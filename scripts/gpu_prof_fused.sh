#!/bin/bash
# ncu --set full of one fused_pass_kernel launch (C2) + the ncu launch list of
# a short bench run + the default bench line.
set -u
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fused_pass -s 2 -c 1 \
  -o gpurun_out/ncu_fused_C2_${TAG} -f python scripts/profile_run.py C2 4096 fused > gpurun_out/ncu_fused_${TAG}.log 2>&1
echo "ncu full exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu_${TAG}.log 2>&1
echo "ncu list exit $?"
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench exit $?"; cat gpurun_out/bench_${TAG}.log
