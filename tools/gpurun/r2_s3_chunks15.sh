# c3 d = 15 (1.2e7 rows) e2e against the pipeline's chunk count (default: rows >> 20 = 11)
for k in 4 6 8 11 16 4 6 8 11 16; do
  TSK_PIPE_CHUNKS=$k timeout 900 python bench.py --config c3 --d 15 --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 d15 chunks $k', 'resp %.2f ms' % (l['response_time_s']*1e3))"
done
