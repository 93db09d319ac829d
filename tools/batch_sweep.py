"""Dev helper: K1 time vs Periodic batch size s on one workload (how much
of K1 scales with batches rather than interactions)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200.engine import search_device

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c5"])
e, q = bench.workload_columns(cfg)
store = tsk.SegmentStore.from_columns(e, validate=False)
queries = tsk.SegmentStore.from_columns(q, validate=False)
del e, q
ix = tsk.build_index(store, 10_000)
for s in [int(v) for v in (sys.argv[2].split(",") if len(sys.argv) > 2 else "30,60,120,240,480,960".split(","))]:
    plan = tsk.periodic(queries, s, ix)
    ints = sum(b.interactions for b in plan.batches)
    r = search_device(store, ix, plan, cfg["d"])
    ks = []
    for _ in range(5):
        r = search_device(store, ix, plan, cfg["d"], queries_resident=True)
        ks.append(r.k1_ms)
    k = float(np.median(ks))
    print(f"s={s}: {len(plan.batches)} batches ints {ints:.4e} k1 {k:.3f} ms -> {ints / k / 1e9:.3f} Tint/s "
          f"({k / len(plan.batches) * 1e3:.2f} us/batch)", flush=True)
