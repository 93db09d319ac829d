"""Dev helper: how a plan's candidate visits split between shared units and
per-batch remainders for pairs and quads (bench configs)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import bench
import paper_1405_7461_b200 as tsk

for name in sys.argv[1:] or ["c5"]:
    cfg = dict(bench.CONFIGS[name])
    e, q = bench.workload_columns(cfg)
    store = tsk.SegmentStore.from_columns(e, validate=False)
    queries = tsk.SegmentStore.from_columns(q, validate=False)
    del e
    ix = tsk.build_index(store, 10_000)
    plan = tsk.periodic(queries, 120, ix)
    fl = np.array([(b.first, b.last) if b.first is not None else (-1, -1) for b in plan.batches], np.int64)
    s = np.array([b.size for b in plan.batches], np.int64)
    for G in (2, 4):
        visits_shared = visits_rem = 0
        for k in range(0, len(s), G):
            f, l, ss = fl[k:k + G, 0], fl[k:k + G, 1], s[k:k + G]
            ilo, ihi = f.max(), l.min()
            if len(ss) >= 2 and (f >= 0).all() and ilo <= ihi and ss.sum() <= 512:
                visits_shared += (ihi - ilo + 1)  # one visit per candidate for the whole group
                visits_rem += ((l - f + 1) - (ihi - ilo + 1)).sum()
            else:
                visits_rem += (l - f + 1).clip(0).sum()
        print(name, f"G={G}: candidate visits shared {visits_shared:.3e}, remainder {visits_rem:.3e}, total {visits_shared + visits_rem:.3e}")
    print(name, "no sharing: visits", (fl[:, 1] - fl[:, 0] + 1).clip(0).sum())
