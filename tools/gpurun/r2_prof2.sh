# profile set for the current kernel: ncu full (c5, c3), launch list (c5 bench), traffic json
TAG=${TAG:-p2}; mkdir -p gpurun_out/$TAG
for c in c5 c3; do
ncu --set full --clock-control none --import-source on -k regex:k1_pairs_f32 -s 3 -c 1 -o gpurun_out/$TAG/k1_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/$TAG/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/$TAG/launches_c5.log 2>&1; echo "launches rc=$?"
