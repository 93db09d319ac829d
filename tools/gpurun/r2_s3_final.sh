# final evidence of the session: GPU suite, smoke, bench lines c1-c5 (CPU baseline + parity), reference arm, c5 ncu launch list
TAG=${TAG:-fin}; mkdir -p gpurun_out/$TAG
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/$TAG/pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/$TAG/smoke.log
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG/bench_c5.json 2> gpurun_out/$TAG/bench_c5.err; echo "c5 rc=$?"
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_ref_c5.json 2> gpurun_out/$TAG/bench_ref_c5.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/$TAG/launches_c5.log 2>&1; echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k1_pairs_f32 -s 3 -c 1 -o gpurun_out/$TAG/k1_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/$TAG/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
