# A/B of K1 variants + host gather probe
nvcc -O3 -o /tmp/hgb tools/host_gather_bench.cu -lpthread 2>/dev/null && /tmp/hgb 85000000 16
VARIANTS="${VARIANTS:-base:variants/libbase.so ffma2:variants/libffma2.so}" CFGS="${CFGS:-c2 c3 c4 c5}" TEST=${TEST:-variants/libffma2.so} bash tools/gpurun/gpurun_ab.sh
