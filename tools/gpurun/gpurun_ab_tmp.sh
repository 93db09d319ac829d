timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
VARIANTS="pair:default base:variants/libv21base.so" CFGS="c1 c2 c3 c4 c5" bash tools/gpurun/gpurun_ab.sh
