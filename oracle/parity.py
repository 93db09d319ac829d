"""Batch-sampled parity of a search result against the C engine oracle —
TEST INFRASTRUCTURE ONLY (tests/ and bench.py's cpu_baseline leg).

Results are plan-invariant and per-batch decomposable
(/root/reference/pkg/src/trajseek/engine.py:176-195),
and the engine's item order is batch order, so the rows of batch b in a
run_search result are a contiguous slice whose offset is the prefix sum of
the per-batch hit counts.  ``check_batches`` evaluates the selected batches
with the C engine (oracle/pair_oracle.c: orc_search_spans) on candidate spans
from the numpy oracle's index (both pinned to the reference's goldens) and
compares every slice bit for bit.
"""

from __future__ import annotations

import time

import numpy as np

from . import c_oracle

RES = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")


def check_batches(store, ix, queries, lo, hi, result_cols, batch_hits, batch_ids, d, *,
                  first=None, last=None, threads=None, batch_overlaps=None):
    """Compare batches ``batch_ids`` of a plan's result with the oracle.

    store / queries: dicts of sorted columns (traj seg xs ys zs ts xe ye ze te);
    ix: numpy-oracle index (or None when first/last are given);
    lo, hi: the plan's batch table; result_cols: the result columns in
    engine order; batch_hits: per-batch hit counts of that result.
    Returns a dict {batches, pairs, hits, mismatches, max_rel_interval_err,
    seconds, spans_equal}; mismatches counts batches whose rows differ.
    """
    t0 = time.perf_counter()
    lo = np.asarray(lo, np.int64)
    hi = np.asarray(hi, np.int64)
    ids = np.asarray(sorted(set(int(b) for b in batch_ids)), np.int64)
    if first is None:
        first, last = c_oracle.plan_spans(store, ix, queries, lo[ids], hi[ids])
    else:
        first = np.asarray(first, np.int64)[ids]
        last = np.asarray(last, np.int64)[ids]
    want, pb = c_oracle.search_spans(store, queries, lo[ids], hi[ids], first, last, d, threads=threads)
    off = np.concatenate([[0], np.cumsum(np.asarray(batch_hits, np.int64))])
    woff = np.concatenate([[0], np.cumsum(pb[:, 0])])
    mism, max_err, pairs = 0, 0.0, 0
    bad = []
    for k, b in enumerate(ids):
        s = slice(int(off[b]), int(off[b + 1]))
        w = slice(int(woff[k]), int(woff[k + 1]))
        if first[k] >= 0:
            pairs += int((last[k] - first[k] + 1) * (hi[b] - lo[b] + 1))
        same = (off[b + 1] - off[b]) == (woff[k + 1] - woff[k])
        if same:
            for c in RES:
                if not np.array_equal(np.asarray(result_cols[c][s]), want[c][w]):
                    same = False
                    break
        if same:
            continue
        mism += 1
        bad.append(int(b))
        n = min(off[b + 1] - off[b], woff[k + 1] - woff[k])
        if n:
            for c in ("t_begin", "t_end"):
                g = np.asarray(result_cols[c][s])[:n]
                h = want[c][w][:n]
                err = np.abs(g - h) / np.maximum(np.abs(h), 1e-300)
                max_err = max(max_err, float(np.nanmax(err)))
    # per-batch temporal overlaps (interactions - temporal misses), when the
    # caller has them (the reference's miss statistics, engine.py:52-55)
    ovl_bad = []
    if batch_overlaps is not None:
        for k, b in enumerate(ids):
            ints = int((last[k] - first[k] + 1) * (hi[b] - lo[b] + 1)) if first[k] >= 0 else 0
            if int(batch_overlaps[b]) != ints - int(pb[k, 1]):
                ovl_bad.append(int(b))
    return {"batches": int(ids.shape[0]), "pairs": pairs, "hits": int(pb[:, 0].sum()),
            "temporal_misses": int(pb[:, 1].sum()), "spatial_misses": int(pb[:, 2].sum()),
            "overlap_mismatches": len(ovl_bad), "bad_overlap_batches": ovl_bad[:10],
            "mismatches": mism, "max_rel_interval_err": max_err, "bad_batches": bad[:10],
            "seconds": time.perf_counter() - t0}
