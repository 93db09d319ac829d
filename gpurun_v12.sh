# v12 FP32 pre-filter: GPU parity, then A/B vs v11
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
VARIANTS="v12:default v11:variants/libv11.so" CFGS="c1 c2 c3 c4 c5" bash gpurun_ab.sh
echo done
