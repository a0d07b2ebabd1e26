#!/bin/bash
# A/B of library builds under variants/<name>/ (plus the in-tree build) on the
# fused batch path: bash scripts/lib_ab.sh name1 name2 ...
for v in "$@"; do
  if [ "$v" = tree ]; then lib=""; else lib="$PWD/variants/$v/libshotsim_b200.so"; fi
  TAG=$v SHOTSIM_B200_LIB=$lib timeout 600 python scripts/fused_bench.py C2:32768 C5:64
done
