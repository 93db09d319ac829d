# v10 filter: GPU parity, then A/B vs the previous kernel and a CPT=3 variant
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
VARIANTS="new:default old:variants/libold.so cpt3:variants/libcpt3.so" CFGS="c3 c5" bash gpurun_ab.sh
echo done
