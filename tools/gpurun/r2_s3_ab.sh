# A/B of library variants on K1 time ($VARIANTS = name:path ..., default = the in-tree build), then the GPU suite
for v in ${VARIANTS:-prev:variants/libprev.so new:default sub64:variants/libsub64.so}; do n=${v%%:*}; l=${v#*:}
  if [ "$l" = default ]; then unset TRAJSEEK_LIB; else export TRAJSEEK_LIB=$PWD/$l; fi
  echo "== $n"; timeout 900 python tools/k1_time.py ${CFGS:-c5 c4 c3} 2>&1 | grep "K1"
done
unset TRAJSEEK_LIB
if [ "${SUITE:-1}" = 1 ]; then timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -2; fi
