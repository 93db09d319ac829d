for v in "tq512:variants/libtq512.so" "t256b:variants/libt256b.so" "def:default"; do
  name=${v%%:*}; lib=${v#*:}
  if [ "$lib" = "default" ]; then unset TRAJSEEK_LIB; else export TRAJSEEK_LIB=$(pwd)/$lib; fi
  for s in 240 120; do
    timeout 900 python bench.py --config c5 --s $s --steps 3 --warmup 2 --no-cpu-baseline --no-parity 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$name s=$s', '%.4g'%d['value'], 'k1 %.2f'%d['roofline']['k1_ms_per_step'], 'ints %.4g'%d['config']['interactions_per_step'])"
  done
done
