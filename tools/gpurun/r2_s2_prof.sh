# round 2 session 2: where time goes — e2e phases (c4, c3), K1 ncu (c5, c3), c5 launch list
mkdir -p gpurun_out/s2p
for c in c4 c3; do TSK_TRACE=1 timeout 600 python tools/e2e_phases.py $c > gpurun_out/s2p/phases_$c.txt 2>&1; echo "phases $c rc=$?"; done
for c in c5 c3; do
ncu --set full --clock-control none --import-source on -k regex:k1_pairs_f32 -s 3 -c 1 -o gpurun_out/s2p/k1_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/s2p/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2p/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/s2p/launches_c5.log 2>&1; echo "launches rc=$?"
