# pipeline: parity tests, then call times on c4/c3
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for c in c4 c3; do echo "== $c"; TSK_TRACE=1 timeout 600 python tools/e2e_phases.py $c 2>&1 | grep "^wall\|pipeline 4" | tail -2 | cut -c1-500; done
for k in 3 4 5 6; do echo "== c4 chunks=$k"; TSK_PIPE_CHUNKS=$k timeout 600 python tools/e2e_phases.py c4 2>&1 | grep "^wall"; done
