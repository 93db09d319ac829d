# quick A/B: GPU suite (optional), benches with parity (no CPU baseline)
# usage: TAG=x SUITE=1 CFGS="c5 c3" bash tools/gpurun/r2_quick.sh
TAG=${TAG:-q}; mkdir -p gpurun_out/$TAG
if [ "${SUITE:-1}" = 1 ]; then timeout 2400 python -m pytest tests -q -m gpu -x 2>&1 | tail -3; fi
for c in ${CFGS:-c5 c4 c3 c2}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_$c.json 2> gpurun_out/$TAG/bench_$c.err; rc=$?
  python - "$c" "$rc" <<'PY'
import json, sys
c, rc = sys.argv[1], sys.argv[2]
try:
    l = json.load(open(f"gpurun_out/{__import__('os').environ.get('TAG','q')}/bench_{c}.json"))
    r = l["roofline"]; p = l.get("parity") or {}
    print(f"{c} rc={rc} value {l['value']:.3e} e2e {l['e2e']['value']:.3e} resp {l['response_time_s']*1e3:.2f}ms k1 {r['k1_ms_per_step']:.2f}ms frac {r['frac']:.3f} evals {r['fp32_prefilter']['evaluated_pairs_per_step']:.3e} parity {p.get('mismatches')}/{p.get('batches')}")
except Exception as e:
    print(c, "rc", rc, "no line", e)
PY
done
