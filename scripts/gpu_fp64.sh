#!/bin/bash
mkdir -p gpurun_out
python scripts/fp64_probe.py > gpurun_out/fp64.log 2>&1
ncu --set full --clock-control none -k regex:fp64_probe -s 1 -c 1 -o gpurun_out/ncu_fp64 -f python scripts/fp64_probe.py >> gpurun_out/fp64.log 2>&1
cat gpurun_out/fp64.log | grep -v "^==PROF"
