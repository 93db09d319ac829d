# A/B: variants given as "name:libpath" in $VARIANTS (path relative to repo root or "default")
[ -n "$LAT" ] && nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp64_latency tools/fp64_latency.cu && /tmp/fp64_latency
for v in $VARIANTS; do
  # name:lib[:ENV=VALUE]
  name=${v%%:*}; rest=${v#*:}; lib=${rest%%:*}; envkv=""
  [ "$rest" != "$lib" ] && envkv=${rest#*:}
  if [ "$lib" = "default" ]; then unset TRAJSEEK_LIB; else export TRAJSEEK_LIB=$(pwd)/$lib; fi
  unset TSK_SPATIAL; [ -n "$envkv" ] && export "$envkv"
  for cfg in ${CFGS:-c5}; do
    out=$(timeout 900 python bench.py --config $cfg --steps ${STEPS:-3} --warmup 2 --no-cpu-baseline --no-parity 2>/tmp/err_$name_$cfg.log)
    echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name', '$cfg', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], 'e2e %.4g'%d['e2e']['value'], 'ms %.2f'%d['ms_per_step'], 'k1 %.2f'%d['roofline']['k1_ms_per_step'])" || tail -5 /tmp/err_$name_$cfg.log
  done
done
unset TSK_SPATIAL
if [ -n "$NCU" ]; then
  export TRAJSEEK_LIB=$(pwd)/${NCU#*:}
  ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 3 -c 1 -o gpurun_out/prof_${NCU%%:*} python bench.py --config ${NCUCFG:-c3} --steps 1 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
  echo ncu done
fi
if [ -n "$TEST" ]; then
  export TRAJSEEK_LIB=$(pwd)/$TEST
  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
fi
