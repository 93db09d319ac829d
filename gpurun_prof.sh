mkdir -p gpurun_out/prof
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 2 -c 1 -o gpurun_out/prof/k1_c5_v14 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out/prof
