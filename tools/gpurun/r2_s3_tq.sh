# A/B: 1024-query tiles (16-warp CTAs, 1 per SM) vs the 512-query default on c5 batch sizes
for v in ${VARIANTS:-base:default tq1024:variants/libtq1024.so}; do n=${v%%:*}; l=${v#*:}
  if [ "$l" = default ]; then unset TRAJSEEK_LIB; else export TRAJSEEK_LIB=$PWD/$l; fi
  echo "== $n"; timeout 900 python tools/batch_sweep.py c5 120,240,480 2>&1 | grep "s="
done
