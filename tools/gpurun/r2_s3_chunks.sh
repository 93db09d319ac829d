# e2e vs pipeline chunk count (TSK_PIPE_CHUNKS; 0 = single launch) on c3 and c4
for c in c3 c4; do for k in ${KS:-0 2 3 4 6 8}; do
  TSK_PIPE_CHUNKS=$k timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c chunks $k', 'e2e %.3e resp %.3f ms  value %.3e' % (l['e2e']['value'], l['response_time_s']*1e3, l['value']))"
done; done
