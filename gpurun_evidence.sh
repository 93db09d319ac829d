# round evidence: full bench line, launch list, ncu full capture of K1 (c5)
mkdir -p gpurun_out/ev
timeout 1200 python bench.py > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev/bench_ref_c5.json 2> gpurun_out/ev/bench_ref_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev/launches_c5.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 2 -c 1 -o gpurun_out/ev/k1_c5 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
nproc > gpurun_out/ev/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/ev/host.txt; free -g >> gpurun_out/ev/host.txt
echo ok
