"""Multi-GPU sharding of a batch plan.

The entry store is replicated in every GPU's HBM; the plan's batches are
cut into contiguous shards with equal total interactions (prefix sum of
``QueryBatch.interactions``, planner.py:61-63).  Batches are independent
and results are plan-invariant (engine.py:176-195), so shards run with no
collective and the combined result is the shard-ordered concatenation —
which is also the reference's item order.
"""

from __future__ import annotations

import numpy as np

from .index import TemporalIndex, candidate_ranges
from .planner import BatchPlan, QueryBatch


def batch_interactions(plan: BatchPlan, index: TemporalIndex) -> np.ndarray:
    """Interactions per batch (engine.py:145 semantics) from the batch extents
    and the index — the same rule the device applies (K3)."""
    lo, hi = plan.table()
    q = plan.queries
    ends = np.maximum.reduceat(q.te, lo)
    f, l = candidate_ranges(index, q.ts[lo], ends)
    return np.where(f >= 0, (l - f + 1) * (hi - lo + 1), 0).astype(np.int64)


# K1's fixed cost per non-empty batch (its work items' set-up, window and
# cull visits) in units of the plan's mean interactions per batch: 1.35 us
# per batch at c5 (Periodic s = 30 vs 120: +10,000 batches, +13.5 ms at equal
# interactions) against ~6e7 interactions per batch at 6.4e-11 ms each.
# Without it the plan's two end shards, whose batches hold fewer candidates,
# ran 9% longer than the middle ones at N = 8 (tools/shard_cost.py).
BATCH_COST_FRAC = 0.35


def shard_bounds(ints: np.ndarray, world: int, batch_cost: float | None = None) -> list[tuple[int, int]]:
    """Contiguous batch shards [b0, b1) with balanced estimated K1 time:
    Σ interactions plus ``batch_cost`` per non-empty batch (default
    ``BATCH_COST_FRAC`` × the mean interactions of a non-empty batch)."""
    nb = int(ints.shape[0])
    ints = np.asarray(ints, dtype=np.float64)
    live = ints > 0
    if batch_cost is None:
        batch_cost = BATCH_COST_FRAC * float(ints[live].mean()) if live.any() else 0.0
    cum = np.concatenate([[0.0], np.cumsum(ints + batch_cost * live, dtype=np.float64)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):  # the batch boundary nearest the target
        t = total * r / world
        i = int(np.searchsorted(cum, t, side="left"))
        if 0 < i <= nb and t - cum[i - 1] <= cum[i] - t:
            i -= 1
        cuts.append(i)
    cuts.append(nb)
    for i in range(1, len(cuts)):
        cuts[i] = min(max(cuts[i], cuts[i - 1]), nb)
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def sub_plan(plan: BatchPlan, b0: int, b1: int) -> BatchPlan | None:
    """Batches [b0, b1) of ``plan`` over a zero-copy view of their queries."""
    if b1 <= b0:
        return None
    bs = plan.batches[b0:b1]
    lo0, hi1 = bs[0].lo, bs[-1].hi
    view = plan.queries.view(lo0, hi1)
    return BatchPlan(view, tuple(QueryBatch(b.lo - lo0, b.hi - lo0, b.extent, b.first, b.last)
                                 for b in bs))
