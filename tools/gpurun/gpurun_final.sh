# final round evidence: bench lines c1-c5, reference arm, launch list, ncu capture, 2-rank smoke, d-sweep, planners,
# sanitizers, the GPU suite with forced batch pairing, perfmodel checks
EV=gpurun_out/ev11 bash tools/gpurun/gpurun_evidence.sh
bash tools/gpurun/gpurun_sanitize.sh
TSK_K1_PAIR=force timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
mkdir -p gpurun_out/pm
timeout 900 python tools/perfmodel_demo.py --config c3 --out gpurun_out/pm/r1_perfmodel_c3.md > /dev/null 2>&1; echo "perfmodel c3 rc=$?"
timeout 900 python tools/perfmodel_demo.py --config c4 --out gpurun_out/pm/r1_perfmodel_c4.md > /dev/null 2>&1; echo "perfmodel c4 rc=$?"
echo all-done
