set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1405_7461_b200._native as n; print(n.probe_fp64(0))"
timeout 300 python __graft_entry__.py smoke
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30
