# 28 B/row (32-bit entry ids, host widening) up to 2^24 rows instead of 2^23: c3 d = 15 (1.2e7 rows) e2e
for v in ids23:variants/libids23.so ids24:variants/libids24.so ids23b:variants/libids23.so ids24b:variants/libids24.so; do n=${v%%:*}; export TRAJSEEK_LIB=$PWD/${v#*:}
  timeout 900 python bench.py --config c3 --d 15 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$n c3 d15', 'e2e %.3e resp %.2f ms parity %s' % (l['e2e']['value'], l['response_time_s']*1e3, l['parity']['mismatches']))"
done
