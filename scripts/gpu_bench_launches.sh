#!/bin/bash
# The default bench line + the ncu launch list of the same command (fewer steps).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?"; cat gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
echo "ncu exit $?"
python profiles/summarize_launches.py gpurun_out/launches_bench.csv
