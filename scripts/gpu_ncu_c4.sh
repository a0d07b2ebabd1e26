timeout 900 ncu --set full --clock-control none -k regex:tile_pass -s 20 -c 1 -o gpurun_out/ncu_c4_pass -f python scripts/profile_run.py C4 256 batch > /dev/null 2>&1; echo ncu $?
timeout 900 ncu --set full --clock-control none -k regex:expval -s 20 -c 1 -o gpurun_out/ncu_c4_expval -f python scripts/profile_run.py C4 256 batch > /dev/null 2>&1; echo ncu2 $?
