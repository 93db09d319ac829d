EV=gpurun_out/ev6 bash tools/gpurun/gpurun_evidence.sh
bash tools/gpurun/gpurun_sanitize.sh
echo all-done
