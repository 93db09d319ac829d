# box-cull radius fix: new absorbed-offset test + extreme goldens, quick benches
mkdir -p gpurun_out/s2b
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "absorbed or extreme" 2>&1 | tail -3
for c in c5 c3 c2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/s2b/bench_$c.json 2> gpurun_out/s2b/bench_$c.err; echo "$c rc=$?"; python -c "
import json;l=json.load(open('gpurun_out/s2b/bench_$c.json'));print('$c', l['value'], l['e2e']['value'], l['roofline']['k1_ms_per_step'])"; done
