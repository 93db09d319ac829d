# round 2 session 2: GPU suite + bench lines (c5 default, c2, c3, c4) with parity
mkdir -p gpurun_out/s2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s2/gpu.txt
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/s2/pytest.log 2>&1; echo "pytest rc=$?"
tail -25 gpurun_out/s2/pytest.log
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/s2/bench_c5.json 2> gpurun_out/s2/bench_c5.err; echo "c5 rc=$?"
for c in c2 c3 c4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/s2/bench_$c.json 2> gpurun_out/s2/bench_$c.err; echo "$c rc=$?"; done
