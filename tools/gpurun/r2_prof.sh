timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
mkdir -p gpurun_out/prof2
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 3 -c 1 -o gpurun_out/prof2/k1_c5_${TAG:-x} python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/prof2/ncu_${TAG:-x}.log 2>&1
echo ncu rc=$?
