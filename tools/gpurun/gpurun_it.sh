# iterate: build, gpu tests, bench c2+c5, ncu c2 K1
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2', d['value'], d['roofline']['frac'], d['e2e']['value'])"
timeout 900 python bench.py --config c5 --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', d['value'], d['roofline']['frac'], d['e2e']['value'], d['ms_per_step'])"
ncu --set full --clock-control none --import-source on -k regex:k1_pairs -s 3 -c 1 -o gpurun_out/prof_c2_$TAG python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
