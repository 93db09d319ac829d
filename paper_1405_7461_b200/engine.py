"""Search execution on the GPU — the drop-in for engine.py.

Same entry points, signatures, statistics and DomainError behaviour as
/root/reference/pkg/src/trajseek/engine.py:

* :func:`execute_batch` (engine.py:97-148) — one batch against an explicit
  candidate span.
* :func:`run_search` (engine.py:151-204) — a whole plan.  All batches go to
  the device in one call: batch extents and candidate ranges (K3), the pair
  kernel over every (batch, candidate tile, query tile) work item (K1), the
  overflow-safe hit buffer, and the radix sort + id gather that returns the
  hits in the reference's order (batch, entry ordinal, query ordinal) (K4).
* :func:`launch_overhead_pass` (engine.py:207-224) — the same launch with
  the pair arithmetic elided.

``workers`` is accepted and validated for API compatibility; parallelism
is the GPU grid.  Per-batch ``kernel_seconds`` cannot be measured inside
one fused launch, so the device time is apportioned by interactions.
"""

from __future__ import annotations

import os
import time
from collections import UserList
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .core import DomainError, ResultSet, SegmentStore
from .index import TemporalIndex
from .planner import BatchPlan


@dataclass
class BatchTrace:
    """Per-batch accounting (engine.py:32-41)."""

    ordinal: int
    queries: int
    candidates: int
    interactions: int
    hits: int
    kernel_seconds: float


@dataclass
class SearchStats:
    """Counters and timings (engine.py:44-66); interactions_computed ==
    temporal_misses + spatial_misses + hits."""

    interactions_computed: int = 0
    temporal_misses: int = 0
    spatial_misses: int = 0
    hits: int = 0
    kernel_seconds: float = 0.0
    overhead_seconds: float = 0.0
    assembly_seconds: float = 0.0
    total_seconds: float = 0.0
    per_batch: list[BatchTrace] = field(default_factory=list)
    # device-side timings (CUDA events): whole pipeline and the K1 launches
    device_seconds: float = 0.0
    pair_kernel_seconds: float = 0.0

    def wasteful_fraction(self) -> float:
        if self.interactions_computed == 0:
            return 0.0
        return (self.temporal_misses + self.spatial_misses) / self.interactions_computed


class _LazyTraces(UserList):
    """``SearchStats.per_batch``: a list of BatchTrace built on first access
    from the per-batch arrays, so a plan of thousands of batches does not pay
    for the Python objects on every call unless they are read.  Every list
    operation goes through ``data``, which fills itself first, so copies,
    concatenation, ``+=``, ``clear``, ``index``, ``sort`` ... all see the
    traces (the reference's per_batch is a plain list, engine.py:56)."""

    def __init__(self, initlist=None, *, src=None):
        self._data = list(initlist) if initlist is not None else []
        self._src = src

    @property
    def data(self):
        if self._src is not None:
            sizes, cands, ints, hits, secs = self._src
            self._src = None
            self._data.extend(map(BatchTrace, range(len(sizes)), sizes, cands, ints, hits, secs))
        return self._data

    @data.setter
    def data(self, value):
        self._src = None
        self._data = value

    def __reduce__(self):
        return (list, (list(self.data),))


def resolve_workers(workers: int | None) -> int:
    """Explicit worker count or machine parallelism (engine.py:69-75)."""
    if workers is None:
        return max(1, os.cpu_count() or 1)
    if workers < 1:
        raise DomainError(f"workers={workers} must be >= 1")
    return workers


def _result_set(res: _native.Result) -> ResultSet:
    c = res.cols
    return ResultSet(c["query_traj"], c["query_seg"], c["entry_traj"], c["entry_seg"],
                     c["t_begin"], c["t_end"])


def execute_batch(store: SegmentStore, batch: SegmentStore, span: tuple[int, int], d: float, *,
                  workers: int | None = None, _noop: bool = False
                  ) -> tuple[ResultSet, SearchStats]:
    """Evaluate one query batch against candidate ordinals span[0]..span[1]."""
    t_start = time.perf_counter()
    resolve_workers(workers)
    first, last = int(span[0]), int(span[1])
    if not (0 <= first <= last < len(store)):
        raise DomainError(f"candidate span {span} outside store of {len(store)} segments")
    if len(batch) == 0:
        raise DomainError("query batch is empty")
    flags = _native.TSK_SPANS_GIVEN | _native.TSK_ORDER_REFERENCE
    if _noop:
        flags |= _native.TSK_NOOP
    res = _native.search(store.device(), batch, [0], [len(batch) - 1], [first], [last], d, flags)
    stats = SearchStats()
    if not _noop:
        ints = (last - first + 1) * len(batch)
        ovl = int(res.per_batch[0, 2])
        stats.interactions_computed = ints
        stats.hits = res.n
        stats.temporal_misses = ints - ovl
        stats.spatial_misses = ovl - res.n
    result = _result_set(res) if res.n else ResultSet.empty()
    stats.device_seconds = res.device_ms / 1e3
    stats.pair_kernel_seconds = res.k1_ms / 1e3
    stats.kernel_seconds = stats.total_seconds = time.perf_counter() - t_start
    return result, stats


def run_search(store: SegmentStore, index: TemporalIndex, plan: BatchPlan, d: float, *,
               workers: int | None = None, devices: list[int] | None = None,
               order: str = "reference") -> tuple[ResultSet, SearchStats]:
    """Execute every batch of ``plan`` against ``store`` on the GPU.

    Additions to the reference signature:

    * ``devices`` shards the plan over several GPUs, each holding a replica
      of the store: contiguous, interaction-balanced batch shards, one host
      thread per device, results concatenated in plan order.
      No collective is involved.
    * ``order="canonical"`` returns the items already in
      ``ResultSet.canonical_order()`` order, sorted on the GPU (K4); the
      default ``"reference"`` is the reference engine's item order.
    """
    resolve_workers(workers)
    if order not in ("reference", "canonical"):
        raise DomainError(f"unknown order {order!r}")
    if devices is not None and len(devices) > 1:
        result, stats = _run_sharded(store, index, plan, d, list(devices))
        return (result.canonical_order() if order == "canonical" else result), stats
    ordinal = None if not devices else devices[0]
    return _run_one(store, index, plan, d, ordinal, 0, order == "canonical")


# Width of K1's hit keys (batch | entry offset | query offset), checked by
# tsk_search; a plan that needs more is run as consecutive sub-plans.
_KEY_BITS = 64


def _bits_for(count: int) -> int:
    """Bits to hold 0..count-1 (search.cu bits_for)."""
    return max(0, int(count - 1).bit_length()) if count > 1 else 0


def _split_for_keys(store, plan):
    """Batch ranges [b0, b1) small enough that each sub-plan's hit keys fit
    in _KEY_BITS bits, or None when the whole plan fits."""
    lo, hi = plan.table()
    eb = _bits_for(max(len(store), 1))
    qb = _bits_for(int((hi - lo + 1).max()))
    if _bits_for(len(plan.batches)) + eb + qb <= _KEY_BITS:
        return None
    room = _KEY_BITS - eb - qb
    if room < 0:
        raise DomainError("a single batch's result keys exceed 64 bits")
    step = 1 << room
    nb = len(plan.batches)
    return [(b0, min(b0 + step, nb)) for b0 in range(0, nb, step)]


def _run_one(store, index, plan, d, ordinal, replica, canonical=False):
    chunks = _split_for_keys(store, plan)
    if chunks is not None:
        return _run_chunked(store, index, plan, d, ordinal, replica, canonical, chunks)
    try:
        return _run_one_call(store, index, plan, d, ordinal, replica, canonical)
    except _native.TooManyHits:
        # more rows than one call returns: halves of the plan, concatenated in
        # plan order (results decompose per batch, engine.py:176-195)
        nb = len(plan.batches)
        if nb < 2:
            raise
        return _run_chunked(store, index, plan, d, ordinal, replica, canonical, [(0, nb // 2), (nb // 2, nb)])


def _run_one_call(store, index, plan, d, ordinal, replica, canonical=False):
    t_start = time.perf_counter()
    queries = plan.queries
    lo, hi = plan.table()
    flags = _native.TSK_ORDER_CANONICAL if canonical else _native.TSK_ORDER_REFERENCE
    res = _indexed_search(store, index, ordinal, replica, queries, lo, hi, d, flags)
    t_asm = time.perf_counter()
    result = _result_set(res) if res.n else ResultSet.empty()
    if canonical:
        result._canonical = True
    stats = SearchStats()
    pb = res.per_batch
    sizes = hi - lo + 1
    cands = np.where(pb[:, 0] >= 0, pb[:, 1] - pb[:, 0] + 1, 0)
    ints = sizes * cands
    total_ints = int(ints.sum())
    dev_s = res.device_ms / 1e3
    share = ints / total_ints if total_ints else np.zeros_like(ints, dtype=np.float64)
    stats.per_batch = _LazyTraces(src=(sizes.tolist(), cands.tolist(), ints.tolist(), pb[:, 3].tolist(),
                                       (share * dev_s).tolist()))
    ovl = int(pb[:, 2].sum())
    stats.interactions_computed = total_ints
    stats.hits = res.n
    stats.temporal_misses = total_ints - ovl
    stats.spatial_misses = ovl - res.n
    stats.kernel_seconds = dev_s
    stats.device_seconds = dev_s
    stats.pair_kernel_seconds = res.k1_ms / 1e3
    t_end = time.perf_counter()
    stats.assembly_seconds = t_end - t_asm
    stats.total_seconds = t_end - t_start
    stats.overhead_seconds = max(0.0, stats.total_seconds - stats.kernel_seconds - stats.assembly_seconds)
    return result, stats


def _indexed_search(store, index, ordinal, replica, queries, lo, hi, d, flags):
    """tsk_search on the device copy carrying ``index``; the handle's lock
    is held from the index check to the end of the search."""
    dev = store.device(ordinal, replica)
    with dev.lock:
        index.ensure_device(ordinal, replica, store)
        return _native.search(dev, queries, lo, hi, None, None, d, flags)


def _run_chunked(store, index, plan, d, ordinal, replica, canonical, chunks):
    """Consecutive sub-plans (keys too wide for one call), concatenated in
    plan order — the reference's item order is per batch, so it is kept."""
    from .sharding import sub_plan

    t_start = time.perf_counter()
    parts, stats = [], SearchStats()
    for b0, b1 in chunks:
        r, st = _run_one(store, index, sub_plan(plan, b0, b1), d, ordinal, replica, False)
        parts.append(r)
        for t in st.per_batch:
            stats.per_batch.append(BatchTrace(t.ordinal + b0, t.queries, t.candidates, t.interactions, t.hits,
                                              t.kernel_seconds))
        for k in ("interactions_computed", "temporal_misses", "spatial_misses", "hits", "kernel_seconds",
                  "device_seconds", "pair_kernel_seconds"):
            setattr(stats, k, getattr(stats, k) + getattr(st, k))
    t_asm = time.perf_counter()
    result = ResultSet.concatenate(parts)
    if canonical:
        result = result.canonical_order()
    t_end = time.perf_counter()
    stats.assembly_seconds = t_end - t_asm
    stats.total_seconds = t_end - t_start
    stats.overhead_seconds = max(0.0, stats.total_seconds - stats.kernel_seconds - stats.assembly_seconds)
    return result, stats


def _run_sharded(store, index, plan, d, devices):
    from concurrent.futures import ThreadPoolExecutor

    from .sharding import batch_interactions, shard_bounds, sub_plan

    t_start = time.perf_counter()
    bounds = shard_bounds(batch_interactions(plan, index), len(devices))
    seen: dict[int, int] = {}
    jobs = []
    for (b0, b1), dvc in zip(bounds, devices):
        replica = seen.get(dvc, 0)
        seen[dvc] = replica + 1
        sp = sub_plan(plan, b0, b1)
        if sp is not None:
            jobs.append((b0, sp, dvc, replica))
    # upload replicas (and their indexes) before the parallel section
    for _, _, dvc, replica in jobs:
        index.ensure_device(dvc, replica, store)
    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as ex:
        outs = list(ex.map(lambda j: _run_one(store, index, j[1], d, j[2], j[3]), jobs))
    stats = SearchStats()
    per_batch: list[BatchTrace] = []
    for (b0, _, _, _), (_, st) in zip(jobs, outs):
        for t in st.per_batch:
            per_batch.append(BatchTrace(t.ordinal + b0, t.queries, t.candidates, t.interactions,
                                        t.hits, t.kernel_seconds))
        stats.interactions_computed += st.interactions_computed
        stats.temporal_misses += st.temporal_misses
        stats.spatial_misses += st.spatial_misses
        stats.hits += st.hits
        stats.kernel_seconds = max(stats.kernel_seconds, st.kernel_seconds)
        stats.device_seconds = max(stats.device_seconds, st.device_seconds)
        stats.pair_kernel_seconds = max(stats.pair_kernel_seconds, st.pair_kernel_seconds)
    # batches of shards that got nothing (more devices than batches) are absent
    # from `jobs`; every batch belongs to exactly one job otherwise
    stats.per_batch = sorted(per_batch, key=lambda t: t.ordinal)
    t_asm = time.perf_counter()
    result = ResultSet.concatenate([r for r, _ in outs])
    t_end = time.perf_counter()
    stats.assembly_seconds = t_end - t_asm
    stats.total_seconds = t_end - t_start
    stats.overhead_seconds = max(0.0, stats.total_seconds - stats.kernel_seconds - stats.assembly_seconds)
    return result, stats


def search_device(store: SegmentStore, index: TemporalIndex, plan: BatchPlan, d: float, *,
                  queries_resident: bool = False) -> _native.Result:
    """Plan execution with hits left in HBM (no D2H of result columns).

    With ``queries_resident`` the query set uploaded by the previous call on
    this store's device copy is reused (no H2D).  Used to time the device
    throughput with inputs resident in HBM; returns the raw result (counts,
    per-batch stats, CUDA-event timings).
    """
    lo, hi = plan.table()
    flags = _native.TSK_ORDER_REFERENCE | _native.TSK_RESULTS_ON_DEVICE
    if queries_resident:
        flags |= _native.TSK_QUERIES_RESIDENT
    return _indexed_search(store, index, None, 0, plan.queries, lo, hi, d, flags)


def launch_overhead_pass(store: SegmentStore, batch: SegmentStore, span: tuple[int, int], *,
                         workers: int | None = None) -> float:
    """Wall seconds of a batch launch with the pair arithmetic elided."""
    _, stats = execute_batch(store, batch, span, 0.0, workers=workers, _noop=True)
    return stats.kernel_seconds


# ── counting passes (perfmodel on the GPU) ──────────────────────────────────


def plan_counts(store: SegmentStore, index: TemporalIndex, plan: BatchPlan, d: float, *,
                overlaps_only: bool = False) -> np.ndarray:
    """Per-batch (first, last, overlaps, hits) of ``plan`` without result rows.

    One fused launch (K3 spans, K1 with no hit rows written).  With
    ``overlaps_only`` K1 skips the geometry and only counts temporally
    overlapping pairs, so ``interactions - overlaps`` is the reference's
    temporal-miss count (perfmodel.py:327-343); hits are then 0.
    """
    lo, hi = plan.table()
    flags = _native.TSK_OVERLAPS_ONLY if overlaps_only else _native.TSK_COUNT_ONLY
    return _indexed_search(store, index, None, 0, plan.queries, lo, hi, d, flags).per_batch


def span_counts(store: SegmentStore, queries: SegmentStore, lo, hi, first, last, d: float, *,
                overlaps_only: bool = False) -> np.ndarray:
    """Per-batch (first, last, overlaps, hits) for explicit batches and spans.

    Batches ``lo[k]..hi[k]`` of ``queries`` (they may overlap each other)
    against candidate ordinals ``first[k]..last[k]``, all in one launch.
    """
    lo = np.ascontiguousarray(lo, dtype=np.int64)
    if lo.shape[0] == 0:
        return np.empty((0, 4), dtype=np.int64)
    flags = _native.TSK_SPANS_GIVEN | (_native.TSK_OVERLAPS_ONLY if overlaps_only else _native.TSK_COUNT_ONLY)
    return _native.search(store.device(), queries, lo, np.ascontiguousarray(hi, dtype=np.int64),
                          np.ascontiguousarray(first, dtype=np.int64),
                          np.ascontiguousarray(last, dtype=np.int64), d, flags).per_batch
