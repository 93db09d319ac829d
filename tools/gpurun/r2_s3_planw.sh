# c4 planners: wide K1 off vs auto (device time, queries resident)
for w in off auto; do for p in periodic setsplit_fixed setsplit_max greedy_min; do
  TSK_K1_WIDE=$w timeout 900 python bench.py --config c4 --planner $p --steps 5 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w $p', 'k1 %.3f device %.3f resp %.3f' % (l['roofline']['k1_ms_per_step'], l['ms_per_step'], l['response_time_s']*1e3))"
done; done
