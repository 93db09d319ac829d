# A/B of library variants on the e2e leg of bench configs ($CFGS), then the pipeline trace of the in-tree build
for v in ${VARIANTS:-prev:variants/libprev.so new:default}; do n=${v%%:*}; l=${v#*:}
  if [ "$l" = default ]; then unset TRAJSEEK_LIB; else export TRAJSEEK_LIB=$PWD/$l; fi
  for c in ${CFGS:-c4}; do
    timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$n $c', 'value %.3e e2e %.3e resp %.2f ms k1 %.2f' % (l['value'], l['e2e']['value'], l['response_time_s']*1e3, l['roofline']['k1_ms_per_step']))"
  done
done
unset TRAJSEEK_LIB
for c in ${CFGS:-c4}; do TSK_TRACE=1 timeout 600 python tools/e2e_phases.py $c 2>&1 | grep -E "pipeline|wall" | tail -3; done
