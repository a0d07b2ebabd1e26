#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py (memcheck, racecheck,
# synccheck, initcheck); logs under gpurun_out/sanitizer_*.log.
set -u
mkdir -p gpurun_out
export SHOTSIM_B200_NO_SPECIALISE=${SHOTSIM_B200_NO_SPECIALISE:-0}
for tool in memcheck synccheck racecheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python scripts/sanitize_run.py \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool exit $?"; tail -3 gpurun_out/sanitizer_$tool.log
done
