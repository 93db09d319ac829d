# wide K1 (16 warps) forced vs off on the smaller configs and on c5's shards: where to switch
for w in off force; do echo "== TSK_K1_WIDE=$w"; TSK_K1_WIDE=$w timeout 600 python tools/k1_time.py c4 c3 c2; done
for w in off force; do echo "== shards TSK_K1_WIDE=$w"; TSK_K1_WIDE=$w timeout 900 python tools/shard_k1.py c5 2>&1 | tail -5; done
