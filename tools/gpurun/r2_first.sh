timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/r2a_c5.err > gpurun_out/r2a_c5.json; tail -c 600 gpurun_out/r2a_c5.json
nproc; lscpu | grep 'Model name'; free -g | head -2
