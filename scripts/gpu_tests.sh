#!/bin/bash
# GPU session: the gpu-marked tests (extra pytest args pass through) + smoke.
# Usage: gpurun --timeout 1800 -- bash scripts/gpu_tests.sh [pytest args...]
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf "$@" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
tail -40 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log
