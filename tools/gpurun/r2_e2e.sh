# e2e breakdown: phases (TSK_TRACE) for $CFGS, host gather probe
mkdir -p gpurun_out/e2e
nvcc -O3 -o /tmp/hgb tools/host_gather_bench.cu -lpthread 2>/dev/null && /tmp/hgb ${HGB_N:-4700000} 16
nproc; lscpu | grep -E "Model name|Socket|NUMA node\(s\)"
for c in ${CFGS:-c4 c3}; do TSK_TRACE=1 timeout 600 python tools/e2e_phases.py $c > gpurun_out/e2e/phases_$c.txt 2>&1; echo "phases $c rc=$?"; grep -E "trace|wall" gpurun_out/e2e/phases_$c.txt | tail -6; done
