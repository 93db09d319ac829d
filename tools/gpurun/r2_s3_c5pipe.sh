# c5 e2e with the pipeline forced to 2 / 3 chunks against the single launch
for k in 0 2 3 0 2 3; do
  TSK_PIPE_CHUNKS=$k timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 chunks $k', 'e2e %.4e resp %.3f ms' % (l['e2e']['value'], l['response_time_s']*1e3))"
done
