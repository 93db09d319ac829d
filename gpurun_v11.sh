# v11 loop restructure: GPU parity, then A/B vs v10
timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
LAT=1 VARIANTS="v11:default v10:variants/libv10.so" CFGS="c3 c4 c5" bash gpurun_ab.sh
echo done
