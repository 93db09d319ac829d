# session 3 re-entry: GPU suite, quick benches, e2e phase breakdown for c3/c4
TAG=s3a SUITE=1 CFGS="c5 c4 c3" bash tools/gpurun/r2_quick.sh 2>&1 | tee gpurun_out/s3a_quick.txt
mkdir -p gpurun_out/s3a
for c in c4 c3; do TSK_TRACE=1 timeout 600 python tools/e2e_phases.py $c > gpurun_out/s3a/phases_$c.txt 2>&1; echo "phases $c rc=$?"; tail -8 gpurun_out/s3a/phases_$c.txt; done
for c in c4 c3; do timeout 600 python tools/host_phases.py $c > gpurun_out/s3a/host_$c.txt 2>&1; echo "host $c rc=$?"; tail -3 gpurun_out/s3a/host_$c.txt; done
