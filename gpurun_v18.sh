timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
VARIANTS="v18:default v17:variants/libv17.so" CFGS="c1 c2 c3 c4 c5" bash gpurun_ab.sh
echo done
