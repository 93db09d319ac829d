"""Temporal-bin index (K2 on the device) and candidate-range lookups (K3).

Same public surface as /root/reference/pkg/src/trajseek/index.py:
``TemporalBin``, ``TemporalIndex``, ``build_index`` (index.py:85-146),
``candidate_range`` (index.py:149-173), ``interaction_count``
(index.py:176-188), ``DEFAULT_BIN_COUNT``.

``build_index`` runs on the GPU: bin assignment with numpy floor-divide
semantics, per-bin first/last ordinals, member/grid extents, per-bin max
end time and its running maximum (libtrajseek ``tsk_index_build``).  The
non-empty-bin arrays are copied back so that host planners can perform the
single-interval lookups of ``candidate_range`` without a device round trip
(the planners are host code); ``run_search``
resolves each batch's range on the device.  Both lookups implement the
same rule, checked against each other and against golden vectors.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import DomainError, SegmentStore, TimeInterval

DEFAULT_BIN_COUNT = 10_000

_EXTENT_RULES = ("member_extents", "grid_start")


@dataclass(frozen=True)
class TemporalBin:
    """A bin's extent and member ordinals; empty bins hold None everywhere."""

    start: float | None
    end: float | None
    first: int | None
    last: int | None

    @property
    def empty(self) -> bool:
        return self.first is None

    @property
    def count(self) -> int:
        return 0 if self.first is None else self.last - self.first + 1


@dataclass(frozen=True, eq=False, repr=False)
class TemporalIndex:
    """Equal-width bins over one store (see index.py:50-82)."""

    m: int
    bin_width: float
    t0: float
    t_max: float
    extent_rule: str
    bins: tuple[TemporalBin, ...]
    _ne_start: np.ndarray
    _ne_end: np.ndarray
    _ne_first: np.ndarray
    _ne_last: np.ndarray
    # running maximum of _ne_end (non-decreasing): first reaching bin by bisection
    _ne_endmax: np.ndarray = None
    _store: SegmentStore = None

    def bin_of(self, t: float) -> int:
        """Index of the bin whose time range contains t."""
        if not self.t0 <= t <= self.t_max:
            raise DomainError(f"t={t!r} outside indexed range [{self.t0!r}, {self.t_max!r}]")
        if self.bin_width == 0.0:
            return 0
        return min(int((t - self.t0) // self.bin_width), self.m - 1)

    def ensure_device(self, ordinal: int | None = None, replica: int = 0, store=None):
        """A device copy of the indexed store (or ``store``) carrying this index."""
        from . import _native

        dev = (self._store if store is None else store).device(ordinal, replica)
        with dev.lock:
            if dev.index_token is not self:
                _native.index_build(dev, self.m, _rule_code(self.extent_rule))
                dev.index_token = self
        return dev


def _rule_code(rule: str) -> int:
    return 0 if rule == "member_extents" else 1


def build_index(store: SegmentStore, m: int = DEFAULT_BIN_COUNT, *,
                extent_rule: str = "member_extents") -> TemporalIndex:
    """Build the m-bin index for ``store`` on the GPU (index.py:85-146)."""
    if m < 1:
        raise DomainError(f"bin count m={m} must be >= 1")
    if extent_rule not in _EXTENT_RULES:
        raise DomainError(f"unknown extent rule {extent_rule!r}; expected one of {_EXTENT_RULES}")
    if len(store) == 0:
        raise DomainError("cannot index an empty store")
    from . import _native

    dev = store.device()
    (width, t0, t_max), ne_start, ne_end, ne_first, ne_last, ne_bin = _native.index_build(
        dev, m, _rule_code(extent_rule))
    bins = [TemporalBin(None, None, None, None)] * m
    for k, j in enumerate(ne_bin.tolist()):
        bins[j] = TemporalBin(float(ne_start[k]), float(ne_end[k]), int(ne_first[k]), int(ne_last[k]))
    ix = TemporalIndex(
        m=int(m), bin_width=float(width), t0=float(t0), t_max=float(t_max),
        extent_rule=extent_rule, bins=tuple(bins),
        _ne_start=ne_start, _ne_end=ne_end, _ne_first=ne_first, _ne_last=ne_last,
        _ne_endmax=np.maximum.accumulate(ne_end) if ne_end.shape[0] else ne_end,
        _store=store,
    )
    dev.index_token = ix
    return ix


def _endmax(index: TemporalIndex) -> np.ndarray:
    em = index._ne_endmax
    if em is None:  # an index assembled by hand
        em = np.maximum.accumulate(index._ne_end) if index._ne_end.shape[0] else index._ne_end
        object.__setattr__(index, "_ne_endmax", em)
    return em


def candidate_range(index: TemporalIndex, q: TimeInterval) -> tuple[int, int] | None:
    """Inclusive candidate ordinals for the closed interval q, or None.

    A bin qualifies when its closed extent meets q; the answer runs from
    the lowest to the highest qualifying bin, bridging gaps (index.py:149-173).
    """
    starts = index._ne_start
    if starts.shape[0] == 0:
        return None
    hi = int(np.searchsorted(starts, q.end, side="right"))
    if hi == 0:
        return None
    k_lo = int(np.searchsorted(_endmax(index)[:hi], q.begin, side="left"))
    if k_lo >= hi:
        return None
    ends = index._ne_end
    k_hi = hi - 1
    while ends[k_hi] < q.begin:
        k_hi -= 1
    return int(index._ne_first[k_lo]), int(index._ne_last[k_hi])


def candidate_ranges(index: TemporalIndex, begin, end) -> tuple[np.ndarray, np.ndarray]:
    """Vectorised candidate ranges of many intervals (first = last = -1 when
    no bin qualifies); same rule as :func:`candidate_range`."""
    begin = np.asarray(begin, dtype=np.float64)
    end = np.asarray(end, dtype=np.float64)
    k = begin.shape[0]
    first = np.full(k, -1, dtype=np.int64)
    last = np.full(k, -1, dtype=np.int64)
    starts = index._ne_start
    if starts.shape[0] == 0 or k == 0:
        return first, last
    hi = np.searchsorted(starts, end, side="right")
    em = _endmax(index)
    k_lo = np.searchsorted(em, begin, side="left")
    ok = (hi > 0) & (k_lo < hi)
    ends = index._ne_end
    k_hi = np.where(ok, hi - 1, 0)
    short = ok & (ends[k_hi] < begin)
    for i in np.nonzero(short)[0]:
        k = int(k_hi[i])
        while ends[k] < begin[i]:
            k -= 1
        k_hi[i] = k
    first[ok] = index._ne_first[k_lo[ok]]
    last[ok] = index._ne_last[k_hi[ok]]
    return first, last


def device_candidate_ranges(index: TemporalIndex, begin, end) -> tuple[np.ndarray, np.ndarray]:
    """:func:`candidate_ranges` evaluated on the GPU (K3, one warp per interval)."""
    from . import _native

    dev = index._store.device()
    with dev.lock:  # the device index must stay this one until the call returns
        index.ensure_device()
        return _native.candidate_ranges(dev, begin, end)


def interaction_count(index: TemporalIndex, batch_size: int, q: TimeInterval) -> int:
    """batch_size × candidate-range size (index.py:176-188)."""
    if batch_size < 0:
        raise DomainError(f"batch_size={batch_size} must be >= 0")
    span = candidate_range(index, q)
    return 0 if span is None else batch_size * (span[1] - span[0] + 1)
