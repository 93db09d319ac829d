"""Index-free search and the exhaustive interaction recount.

Same API as /root/reference/pkg/src/trajseek/oracle.py (the reference's
validation helpers, re-exported from its package root):

* :func:`brute_force_search` (oracle.py:23-41) — every query against every
  entry, query-major order; runs on the GPU as one batch spanning the
  whole store with (query, entry) result keys.
* :func:`count_interactions_naive` (oracle.py:44-70) — per-batch counts by
  scanning every bin without the contiguity shortcut (host).
"""

from __future__ import annotations

from . import _native
from .core import ResultSet, SegmentStore
from .index import TemporalIndex
from .planner import BatchPlan


def brute_force_search(store: SegmentStore, queries: SegmentStore, d: float) -> ResultSet:
    """All hits, query-major (query ordinal, then entry ordinal)."""
    if len(store) == 0 or len(queries) == 0:
        from .core import pair_intervals

        pair_intervals(queries, store, d)  # argument validation only
        return ResultSet.empty()
    flags = _native.TSK_SPANS_GIVEN | _native.TSK_ORDER_QUERY_MAJOR
    res = _native.search(store.device(), queries, [0], [len(queries) - 1], [0], [len(store) - 1],
                         d, flags)
    if res.n == 0:
        return ResultSet.empty()
    c = res.cols
    return ResultSet(c["query_traj"], c["query_seg"], c["entry_traj"], c["entry_seg"],
                     c["t_begin"], c["t_end"])


def count_interactions_naive(index: TemporalIndex, plan: BatchPlan) -> list[int]:
    """Per-batch interactions from a scan over every bin (oracle.py:44-70)."""
    out = []
    live = [b for b in index.bins if not b.empty]
    for batch in plan.batches:
        q = batch.extent
        hits = [b for b in live if b.start <= q.end and b.end >= q.begin]
        if not hits:
            out.append(0)
            continue
        lo = min(b.first for b in hits)
        hi = max(b.last for b in hits)
        out.append(batch.size * (hi - lo + 1))
    return out
