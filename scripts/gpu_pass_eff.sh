#!/bin/bash
# Per-pass FP64 efficiency of C2 (launch list, trunk off) + one full ncu capture with SASS.
set -u
mkdir -p gpurun_out
CFG=${1:-C2}; SHOTS=${2:-2048}
python scripts/profile_run.py $CFG 64 > /dev/null 2>&1   # warm the NVRTC cache outside ncu
SHOTSIM_B200_NO_TRUNK=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/pe_${CFG}.csv python scripts/profile_run.py $CFG $SHOTS > gpurun_out/pe_${CFG}.log 2>&1
python scripts/pass_efficiency.py $CFG $SHOTS gpurun_out/pe_${CFG}.csv | tee gpurun_out/pe_${CFG}.txt
SHOTSIM_B200_NO_TRUNK=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:tile_pass -s ${3:-2} -c 1 \
  -o gpurun_out/ncu_${CFG}_src -f python scripts/profile_run.py $CFG $SHOTS > gpurun_out/ncu_${CFG}_src.log 2>&1
tail -2 gpurun_out/ncu_${CFG}_src.log
