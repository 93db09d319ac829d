"""Dev helper: host-side time of the phases of one run_search on a small config."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200 import _native, engine

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"])
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
ix = tsk.build_index(store, 10_000)
plan = tsk.periodic(queries, 120, ix)
pq = tsk.SegmentStore(*(_native.pinned_copy(np.ascontiguousarray(getattr(queries, k))) for k in bench.FIELDS),
                      validate=False, presorted=True)
plan = tsk.BatchPlan(pq, plan.batches)
d = cfg["d"]
for _ in range(5):
    tsk.run_search(store, ix, plan, d)
acc = {}
def tick(name, t0):
    acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
    return time.perf_counter()
N = 50
for _ in range(N):
    t = time.perf_counter()
    lo, hi = plan.table(); t = tick("table", t)
    dev = ix.ensure_device(None, 0, store); t = tick("ensure_device", t)
    col, keep = _native.columns_of(pq); t = tick("columns_of", t)
    res = _native.search(dev, pq, lo, hi, None, None, d, _native.TSK_ORDER_REFERENCE); t = tick("tsk_search+Result", t)
    rs = engine._result_set(res); t = tick("ResultSet", t)
T = time.perf_counter()
for _ in range(N):
    tsk.run_search(store, ix, plan, d)
full = (time.perf_counter() - T) / N
print({k: round(v / N * 1e6, 1) for k, v in acc.items()}, "us;  run_search", round(full * 1e6, 1), "us; device",
      round(res.device_ms * 1e3, 1), "us")
