#!/bin/bash
# GPU parity tests + per-config timings (+ optional bench).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/config_timing.py > gpurun_out/timing.log 2>&1; echo "timing exit $?" >> gpurun_out/timing.log
if [ "${1:-}" = "bench" ]; then timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log; fi
tail -5 gpurun_out/pytest_gpu.log; cat gpurun_out/timing.log; cat gpurun_out/bench.log 2>/dev/null
