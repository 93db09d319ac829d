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


def shard_bounds(ints: np.ndarray, world: int) -> list[tuple[int, int]]:
    """Contiguous batch shards [b0, b1) with balanced Σ interactions."""
    nb = int(ints.shape[0])
    cum = np.concatenate([[0.0], np.cumsum(ints, dtype=np.float64)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
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
