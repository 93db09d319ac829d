# parity on EVERY batch of the bench configs (TSK_PARITY_BATCHES above the batch count; the C engine oracle on the host cores)
TAG=${TAG:-fp}; mkdir -p gpurun_out/$TAG
for c in c5 c4 c3 c2; do
  TSK_PARITY_BATCHES=100000 timeout 2400 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; echo "$c rc=$?"
  grep "\[parity\]" gpurun_out/$TAG/bench_$c.err
done
TSK_PARITY_BATCHES=100000 timeout 2400 python bench.py --config c3 --d 30 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c3_d30.json 2> gpurun_out/$TAG/bench_c3_d30.err; echo "c3 d30 rc=$?"
grep "\[parity\]" gpurun_out/$TAG/bench_c3_d30.err
