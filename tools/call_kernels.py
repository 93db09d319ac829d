"""Dev helper: two run_search calls of a bench config (the second is the
one to read), for a per-launch ncu list:
  ncu --metrics gpu__time_duration.sum --csv python tools/call_kernels.py c4"""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200 import _native

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"])
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
ix = tsk.build_index(store, 10_000)
plan = tsk.periodic(queries, 120, ix)
pq = tsk.SegmentStore(*(_native.pinned_copy(np.ascontiguousarray(getattr(queries, k))) for k in bench.FIELDS),
                      validate=False, presorted=True)
plan = tsk.BatchPlan(pq, plan.batches)
for _ in range(2):
    tsk.run_search(store, ix, plan, cfg["d"])
