# round evidence: full bench line, reference arm, launch list, ncu full capture of K1 (c5), 2-rank smoke
mkdir -p gpurun_out/ev3
timeout 1200 python bench.py > gpurun_out/ev3/bench_c5.json 2> gpurun_out/ev3/bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev3/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 2 -c 1 -o gpurun_out/ev3/k1_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
TSK_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --steps 3 --warmup 2 > gpurun_out/ev3/bench_c3_2rank_samegpu.json 2> gpurun_out/ev3/bench_c3_2rank.err
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/ev3/bench_$c.json 2> gpurun_out/ev3/bench_$c.err; done
echo ok
