# chunk sorts beside K1: reserved SMs sweep on c4 e2e; warp-decode K1 variant A/B
for m in 16 32 48; do
  TSK_PIPE_SORT_SMS=$m timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline --no-parity 2>/dev/null | python -c "
import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sms $m c4', 'e2e %.3e resp %.2f ms' % (l['e2e']['value'], l['response_time_s']*1e3))"
  TSK_PIPE_SORT_SMS=$m TSK_TRACE=1 timeout 600 python tools/e2e_phases.py c4 2>&1 | grep -E "pipeline [0-9]" | tail -1
done
VARIANTS="base:default wdec:variants/libwdec.so" SUITE=0 CFGS="c5 c4 c3" bash tools/gpurun/r2_s3_ab.sh
TRAJSEEK_LIB=$PWD/variants/libwdec.so timeout 900 python -m pytest tests -q -m gpu -x -k "octets or quads or config" 2>&1 | tail -1
