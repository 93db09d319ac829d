# round 2: GPU suite (incl. scale parity), bench lines with parity + honest roofline
mkdir -p gpurun_out/r2p
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 2>&1 | tail -25
for c in c1 c2; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/r2p/bench_$c.json 2> gpurun_out/r2p/bench_$c.err; echo "$c rc=$?"; done
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r2p/bench_c5.json 2> gpurun_out/r2p/bench_c5.err; echo "c5 rc=$?"
tail -3 gpurun_out/r2p/bench_c5.err
