#!/bin/bash
# Full GPU validation + per-config report with clocks (round 2).
set -u
mkdir -p gpurun_out
bash scripts/gpu_tests.sh "$@"
timeout 900 python scripts/config_report.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs exit $?"
cat gpurun_out/configs.jsonl
