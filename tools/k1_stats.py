"""Dev helper: K1 development counters for one search of a bench config.
Needs a library built with -DTSK_K1_STATS (TRAJSEEK_LIB=...)."""
import sys
sys.path.insert(0, ".")
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200 import _native

for name in sys.argv[1:] or ["c5"]:
    cfg = dict(bench.CONFIGS[name])
    e, q = bench.workload_columns(cfg)
    store = tsk.SegmentStore.from_columns(e, validate=False)
    queries = tsk.SegmentStore.from_columns(q, validate=False)
    del e, q
    ix = tsk.build_index(store, 10_000)
    plan = tsk.periodic(queries, 120, ix)
    tsk.run_search(store, ix, plan, cfg["d"])
    _native.k1_stats(reset=True)
    res, st = tsk.run_search(store, ix, plan, cfg["d"])
    s = _native.k1_stats()
    print(name, "interactions", st.interactions_computed, "hits", st.hits, s, flush=True)
