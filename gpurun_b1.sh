python -c "import __graft_entry__ as g; g.build()" 
timeout 600 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline
