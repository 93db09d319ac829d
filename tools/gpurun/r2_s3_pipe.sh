# chunk sorts beside K1 vs serial: pipeline tests, c4 and c3 (d = 15) e2e, traces
timeout 1500 python -m pytest tests -q -m gpu -x -k "pipe or chunk or overflow or beyond or split or c4 or scale" 2>&1 | tail -2
for m in serial beside; do
  for c in c4; do
    TSK_PIPE_SORT=$m timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$m $c', 'value %.3e e2e %.3e resp %.2f ms k1 %.2f parity %s' % (l['value'], l['e2e']['value'], l['response_time_s']*1e3, l['roofline']['k1_ms_per_step'], l['parity']['mismatches']))"
  done
  TSK_PIPE_SORT=$m TSK_TRACE=1 timeout 600 python tools/e2e_phases.py c4 2>&1 | grep -E "pipeline [0-9]" | tail -1
  TSK_PIPE_SORT=$m timeout 900 python tools/e2e_phases.py c3 15 2>&1 | grep -E "wall" | tail -1
done
