"""Dev helper: K1 time of one rank's shard of c5 at N = 1, 2, 4, 8 (the
scaling run's per-rank work), on this one GPU."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200.engine import search_device
from paper_1405_7461_b200.sharding import shard_bounds, sub_plan

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"])
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
del e, q
ix = tsk.build_index(store, 10_000)
plan = tsk.periodic(queries, 120, ix)
ints = np.array([b.interactions for b in plan.batches], np.int64)
t1 = None
for world in (1, 2, 4, 8):
    dev = []
    for rank, (b0, b1) in enumerate(shard_bounds(ints, world)):
        sp = sub_plan(plan, b0, b1)
        r = search_device(store, ix, sp, cfg["d"])
        ds = []
        for _ in range(5):
            r = search_device(store, ix, sp, cfg["d"], queries_resident=True)
            ds.append(r.device_ms)
        dev.append(float(np.median(ds)))
    t = max(dev)
    t1 = t if world == 1 else t1
    print(f"N={world}: per-rank device ms {[round(x, 2) for x in dev]}, max {t:.3f} -> "
          f"{ints.sum() / (t / 1e3):.3e} pair-evals/s, efficiency {t1 / (world * t):.3f}", flush=True)
