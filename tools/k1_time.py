"""Dev helper: median K1 and device time (queries resident) of bench configs,
for A/B runs of library variants (TRAJSEEK_LIB=...)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200.engine import search_device

for name in sys.argv[1:] or ["c5"]:
    cfg = dict(bench.CONFIGS[name])
    e, q = bench.workload_columns(cfg)
    store = tsk.SegmentStore.from_columns(e, validate=False)
    queries = tsk.SegmentStore.from_columns(q, validate=False)
    del e, q
    ix = tsk.build_index(store, 10_000)
    plan = tsk.periodic(queries, 120, ix)
    r = search_device(store, ix, plan, cfg["d"])
    ks, ds = [], []
    for _ in range(15):
        r = search_device(store, ix, plan, cfg["d"], queries_resident=True)
        ks.append(r.k1_ms)
        ds.append(r.device_ms)
    print(f"{name}: K1 {np.median(ks):.3f} ms (min {min(ks):.3f}), device {np.median(ds):.3f} ms, hits {r.n}", flush=True)
    del store, queries, ix, plan
