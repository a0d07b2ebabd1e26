#!/bin/bash
# ncu --set full captures of the SM-resident kernels: resident_kernel (C1
# one-warp build, C3 CTA build) and b_child_run_kernel (C3 branch).
set -u
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident_kernel -c 1 \
  -o gpurun_out/ncu_C1_resident -f python scripts/profile_run.py C1 1000000 batch > gpurun_out/ncu_C1.log 2>&1; echo "C1 $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:resident_kernel -c 1 \
  -o gpurun_out/ncu_C3_resident -f python scripts/profile_run.py C3 200000 batch > gpurun_out/ncu_C3r.log 2>&1; echo "C3r $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:b_child_run -s 6 -c 1 \
  -o gpurun_out/ncu_C3_child -f python scripts/profile_run.py C3 1000000 branch:65536 > gpurun_out/ncu_C3b.log 2>&1; echo "C3b $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3b.csv \
  python scripts/profile_run.py C3 1000000 branch:65536 > /dev/null 2>&1; echo "C3 list $?"
