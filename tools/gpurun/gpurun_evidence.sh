# round evidence: bench lines c1-c5, reference arm, launch list, ncu full capture of K1 (c5), 2-rank smoke, d sweep, planners
EV=${EV:-gpurun_out/ev4}
mkdir -p $EV gpurun_out/ds gpurun_out/pl
timeout 1200 python bench.py > $EV/bench_c5.json 2> $EV/bench_c5.err; tail -c 300 $EV/bench_c5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $EV/bench_ref_c5.json 2> $EV/bench_ref_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $EV/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 2 -c 1 -o $EV/k1_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
TSK_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --steps 3 --warmup 2 > $EV/bench_c3_2rank_samegpu.json 2> $EV/bench_c3_2rank.err
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $EV/bench_$c.json 2> $EV/bench_$c.err; done
[ -z "$SKIP_SWEEPS" ] && bash tools/gpurun/gpurun_dsweep.sh
[ -z "$SKIP_SWEEPS" ] && bash tools/gpurun/gpurun_planners.sh
echo ok
