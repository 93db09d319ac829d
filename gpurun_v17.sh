timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
VARIANTS="v17:default v15:variants/libv15b.so" CFGS="c2 c3 c4 c5" bash gpurun_ab.sh
echo done
