# 1q Kraus probability kernel (g_expval1_staged): pairs per thread per staged round (shared memory per
# CTA and CTAs per SM), on C4 (exact batch).
for v in tree e1p8 e1p4 tree e1p8 e1p4; do
  if [ $v = tree ]; then L=""; else L=$PWD/variants/$v/libshotsim_b200.so; fi
  TAG=$v SHOTSIM_B200_LIB=$L timeout 600 python scripts/exact_bench.py C4:256 2>&1 | tail -1
done
