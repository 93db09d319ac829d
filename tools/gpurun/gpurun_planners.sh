mkdir -p gpurun_out/pl
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for p in periodic setsplit_fixed setsplit_max setsplit_minmax greedy_min greedy_max; do
  timeout 900 python bench.py --config c4 --planner $p --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/pl/c4_$p.json 2> gpurun_out/pl/c4_$p.err
done
echo ok
