#!/bin/bash
# ncu capture of the dominant kernel (one launch) + per-config timings.
# Usage: gpurun --timeout 1500 -- bash scripts/gpu_prof.sh [config] [shots] [tag]
set -u
CFG=${1:-C2}; SHOTS=${2:-2048}; TAG=${3:-cur}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/config_timing.py > gpurun_out/timing.log 2>&1; echo "timing exit $?" >> gpurun_out/timing.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tile_pass_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_${CFG}_${TAG} -f python scripts/profile_run.py $CFG $SHOTS > gpurun_out/ncu_${CFG}_${TAG}.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_${CFG}_${TAG}.log
tail -2 gpurun_out/pytest_gpu.log; cat gpurun_out/timing.log; tail -3 gpurun_out/ncu_${CFG}_${TAG}.log
