# round-2 evidence for the current kernel: GPU suite, bench lines c1-c5 (with CPU
# baseline + parity), reference arm at c5, ncu full (c5, c3), c5 launch list
TAG=${TAG:-ev}; mkdir -p gpurun_out/$TAG
timeout 2400 python -m pytest tests -q -m gpu -x > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/$TAG/pytest.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$TAG/gpu.txt
nproc > gpurun_out/$TAG/host.txt; lscpu | grep -E "Model name|Socket" >> gpurun_out/$TAG/host.txt; free -g | head -2 >> gpurun_out/$TAG/host.txt
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/$TAG/bench_c5.json 2> gpurun_out/$TAG/bench_c5.err; echo "c5 rc=$?"
for c in c1 c2 c3 c4; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; echo "$c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/$TAG/bench_ref_c5.json 2> gpurun_out/$TAG/bench_ref_c5.err; echo "ref rc=$?"
TAG=$TAG bash tools/gpurun/r2_prof2.sh
# 2 ranks on the one GPU (TSK_BENCH_DEVICE pins both; timing collectives over gloo): the N>1 path end to end
TSK_BENCH_DEVICE=0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c3 --steps 5 --warmup 3 > gpurun_out/$TAG/bench_c3_2rank_samegpu.json 2> gpurun_out/$TAG/bench_c3_2rank.err; echo "2rank rc=$?"
