# ncu --set full of K1 for the configs in $CFGS, tag $TAG
TAG=${TAG:-n}; mkdir -p gpurun_out/$TAG
for c in ${CFGS:-c5}; do
ncu --set full --clock-control none --import-source on -k regex:k1_pairs_f32 -s 3 -c 1 -o gpurun_out/$TAG/k1_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline --no-parity > gpurun_out/$TAG/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
