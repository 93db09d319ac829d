timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
TEST=variants/libmb3.so bash gpurun_ab.sh
VARIANTS="mb2:default mb3:variants/libmb3.so mb4:variants/libmb4.so v13:variants/libv13.so" CFGS="c3 c5" bash gpurun_ab.sh
echo done
