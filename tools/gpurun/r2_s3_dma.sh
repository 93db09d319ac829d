# pinned query columns: copy-engine upload + device query kernel (TSK_QUERY_DMA) against the kernel reading mapped host memory
export TRAJSEEK_LIB=$PWD/variants/libdma.so
for m in mapped dma mapped dma; do
  if [ $m = dma ]; then export TSK_QUERY_DMA=1; else unset TSK_QUERY_DMA; fi
  for c in c5 c3; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m $c', 'e2e %.4e resp %.3f ms' % (l['e2e']['value'], l['response_time_s']*1e3))"
  done
done
TSK_QUERY_DMA=1 TSK_TRACE=1 timeout 600 python tools/e2e_phases.py c5 2>&1 | grep -E "trace" | tail -1
