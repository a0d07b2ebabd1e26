# Exact tile pass single- vs double-buffered (SHOTSIM_B200_TILE_DB, NVRTC build): C4 at tiles 11 / 12,
# C2 / C5 exact at the default tile; values compared inside each script.
for db in 0 1 0 1; do
  SHOTSIM_B200_TILE_DB=$db TAG=db$db timeout 600 python scripts/exact_bench.py C4:256 C2:16384 C5:32 2>&1 | tail -3
done
for db in 0 1; do
  SHOTSIM_B200_TILE_DB=$db timeout 600 python scripts/probes/c4_tiles.py 256 2>&1 | head -2 | sed "s/^/db$db /"
done
