# v10 filter: GPU parity, then A/B vs the previous kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
VARIANTS="new:default old:variants/libold.so" CFGS="c3 c4 c5" bash gpurun_ab.sh
echo done
