# octets / wide K1: parity suite, then K1 time with the wide kernel off / auto / forced
timeout 1500 python -m pytest tests -q -m gpu -x -k "${K:-}" 2>&1 | tail -4
for w in off auto; do echo "== TSK_K1_WIDE=$w"; TSK_K1_WIDE=$w timeout 900 python tools/k1_time.py ${CFGS:-c5 c4 c3}; done
echo "== TSK_K1_WIDE=force"; TSK_K1_WIDE=force timeout 900 python tools/k1_time.py ${FCFGS:-c4 c3}
