# Exact tile pass with / without the L2 prefetch of the next tile (NVRTC knob).
for pf in 1 0 1 0; do
  SHOTSIM_B200_TILE_PREFETCH=$pf TAG=prefetch$pf timeout 600 python scripts/exact_bench.py C4:256 C2:16384 C5:32 2>&1 | tail -3
done
