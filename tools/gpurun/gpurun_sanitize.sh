mkdir -p gpurun_out/san
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "unsorted or resident" 2>&1 | tail -2
timeout 900 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san/memcheck.txt 2>&1; echo "memcheck rc=$?"
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san/racecheck.txt 2>&1; echo "racecheck rc=$?"
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san/synccheck.txt 2>&1; echo "synccheck rc=$?"
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/san/initcheck.txt 2>&1; echo "initcheck rc=$?"
tail -3 gpurun_out/san/*.txt
