# SURVEY §8d workload coverage with the final kernel: c2 at the S1/S2 analogue
# thresholds (d = 0.15, 1.0) x Periodic s in {60, 120, 240}; c3 Normal and
# Normal5 d-sweeps {1, 5, 15, 30}; c4 under the six planners.  Bench lines
# with parity (no CPU baseline), one JSON file per run.
TAG=${TAG:-sw}; mkdir -p gpurun_out/$TAG
run() { timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/$TAG/$(echo "$@" | tr ' ' '_' | tr -d '-').json 2>> gpurun_out/$TAG/err.log; echo "$* rc=$?"; }
for d in 0.15 1.0; do for s in 60 120 240; do run --config c2 --d $d --s $s; done; done
for c in c3 c3n5; do for d in 1 5 15 30; do run --config $c --d $d; done; done
for p in periodic setsplit_fixed setsplit_max setsplit_minmax greedy_min greedy_max; do run --config c4 --planner $p; done
