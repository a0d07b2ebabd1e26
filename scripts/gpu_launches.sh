#!/bin/bash
# ncu launch list (per-kernel durations) of one config run: gpurun -- bash scripts/gpu_launches.sh C4 64
CFG=${1:-C4}; SHOTS=${2:-64}; MODE=${3:-batch}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${CFG}_${MODE}.csv \
  python scripts/profile_run.py $CFG $SHOTS $MODE > gpurun_out/launches_${CFG}_${MODE}.log 2>&1
python profiles/summarize_launches.py gpurun_out/launches_${CFG}_${MODE}.csv
