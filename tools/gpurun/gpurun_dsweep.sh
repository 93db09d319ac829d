mkdir -p gpurun_out/ds
for d in 1 5 15 30 50; do
  timeout 900 python bench.py --config c3 --d $d --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ds/c3_d$d.json 2> gpurun_out/ds/c3_d$d.err || tail -3 gpurun_out/ds/c3_d$d.err
done
TSK_TRACE=1 timeout 600 python bench.py --config c3 --d 50 --steps 1 --warmup 1 --no-cpu-baseline 2>&1 >/dev/null | grep "tsk trace" | tail -2
echo ok
