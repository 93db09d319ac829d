timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
VARIANTS="v15:default v14:variants/libv14.so" CFGS="c1 c2 c3 c4 c5" bash gpurun_ab.sh
echo done
