# one ncu --set full capture of K1 (c5 and c3) + the new GPU tests
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "fp32 or filter" 2>&1 | tail -2
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 2 -c 1 -o gpurun_out/prof/k1_c5_v12 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 3 -c 1 -o gpurun_out/prof/k1_c3_v12 python bench.py --config c3 --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/prof
