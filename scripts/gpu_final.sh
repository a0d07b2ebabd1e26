#!/bin/bash
# Round-end evidence: bench line, ncu launch list of the bench command, one
# ncu --set full of the dominant kernel, per-config report with clocks.
set -u
mkdir -p gpurun_out
TAG=${1:-r02}
timeout 1200 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; echo "bench exit $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_ncu_${TAG}.log 2>&1; echo "ncu list exit $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:fused_pass -s 3 -c 1 \
  -o gpurun_out/ncu_fused_${TAG} -f python scripts/profile_run.py C2 4096 fused > /dev/null 2>&1; echo "ncu full exit $?"
timeout 1500 python scripts/config_report.py > gpurun_out/configs_${TAG}.jsonl 2> gpurun_out/configs_${TAG}.err; echo "configs exit $?"
cat gpurun_out/bench_${TAG}.log gpurun_out/configs_${TAG}.jsonl
