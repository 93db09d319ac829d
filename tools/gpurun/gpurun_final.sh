# final round evidence: bench lines c1-c5, reference arm, launch list, ncu capture, 2-rank smoke, d-sweep, planners, sanitizers
EV=gpurun_out/ev9 bash tools/gpurun/gpurun_evidence.sh
bash tools/gpurun/gpurun_sanitize.sh
echo all-done
