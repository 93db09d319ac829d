"""Dev helper: where does run_search's host time go on a small config?"""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200 import _native

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"])
if len(sys.argv) > 2:
    cfg["d"] = float(sys.argv[2])
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
ix = tsk.build_index(store, 10_000)
plan = tsk.periodic(queries, 120, ix)
pq = tsk.SegmentStore(*(_native.pinned_copy(np.ascontiguousarray(getattr(queries, k))) for k in bench.FIELDS),
                      validate=False, presorted=True)
plan = tsk.BatchPlan(pq, plan.batches)
for _ in range(3):
    tsk.run_search(store, ix, plan, cfg["d"])
ts = []
for _ in range(4):
    t = time.perf_counter(); r, st = tsk.run_search(store, ix, plan, cfg["d"]); ts.append(time.perf_counter() - t)
    print("call ms", ts[-1] * 1e3, "device ms", st.device_seconds * 1e3, flush=True)
print("wall ms", np.median(ts) * 1e3, "device ms", st.device_seconds * 1e3, "k1 ms", st.pair_kernel_seconds * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    tsk.run_search(store, ix, plan, cfg["d"])
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
