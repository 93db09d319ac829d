"""Dev helper: per-shard cost drivers at N ranks (interactions, queries,
candidates, overlaps, hits) beside the shard's K1 and device time."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200.engine import search_device
from paper_1405_7461_b200.sharding import shard_bounds, sub_plan

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"])
world = int(sys.argv[2]) if len(sys.argv) > 2 else 8
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
del e, q
ix = tsk.build_index(store, 10_000)
plan = tsk.periodic(queries, 120, ix)
ints = np.array([b.interactions for b in plan.batches], np.int64)
rows = []
for rank, (b0, b1) in enumerate(shard_bounds(ints, world)):
    sp = sub_plan(plan, b0, b1)
    r = search_device(store, ix, sp, cfg["d"])
    ks, ds = [], []
    for _ in range(5):
        r = search_device(store, ix, sp, cfg["d"], queries_resident=True)
        ks.append(r.k1_ms); ds.append(r.device_ms)
    pb = np.asarray(r.per_batch)
    lo, hi = sp.table()
    nq = int((hi - lo + 1).sum()); nc = int(np.where(pb[:, 0] >= 0, pb[:, 1] - pb[:, 0] + 1, 0).sum())
    print(f"rank {rank}: {b1 - b0} batches ints {ints[b0:b1].sum():.4e} q {nq} cand {nc} ovl {int(pb[:, 2].sum()):.4e} "
          f"hits {int(pb[:, 3].sum()):.4e} k1 {np.median(ks):.3f} dev {np.median(ds):.3f}", flush=True)
