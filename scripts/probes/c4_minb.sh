# C4 exact tile pass: CTAs per SM (JIT launch bound) x tile size.
for mb in 3 4 5 6; do
  SHOTSIM_B200_JIT_MINB=$mb timeout 600 python scripts/probes/c4_tiles.py 256 2>&1 | head -2 | sed "s/^/minb$mb /"
done
