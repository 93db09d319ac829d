timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
VARIANTS="${VARIANTS:-sub8:default sub16:variants/libsub16.so sub32:variants/libsub32.so}" CFGS="${CFGS:-c5 c4 c3 c2}" STEPS=5 bash tools/gpurun/gpurun_ab.sh
TSK_TRACE=1 timeout 600 python tools/e2e_phases.py c4 2>&1 | grep -E "trace|wall" | tail -3
