timeout 1800 python -m pytest tests -q -m gpu -x 2>&1 | tail -5
VARIANTS="${VARIANTS:-fast:default cull:default:TSK_SPATIAL=noext}" CFGS="${CFGS:-c2 c3 c4 c5}" TEST= bash tools/gpurun/gpurun_ab.sh
