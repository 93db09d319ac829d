"""Randomized properties of K1 (through pair_intervals), after the reference's
hypothesis tests (/root/reference/pkg/tests/test_core.py:163-225): symmetry
in the operands, monotonicity in d, intervals inside the shared span — plus
equality with the C oracle on every drawn example.  Many pairs go to the GPU
per example (a row x column mesh), so each property sees thousands of pairs.
"""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_1405_7461_b200 as tsk
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

coord = st.floats(-50.0, 50.0, allow_nan=False, allow_infinity=False)
time_val = st.floats(0.0, 20.0, allow_nan=False, allow_infinity=False)
span_val = st.floats(0.0, 5.0, allow_nan=False, allow_infinity=False)
dist = st.floats(0.0, 30.0, allow_nan=False, allow_infinity=False)


@st.composite
def meshes(draw):
    """Rows and columns anchored at a few shared start times (extents overlap
    often, and exactly-equal times are common), 1-6 by 1-6 segments."""
    anchors = draw(st.lists(time_val, min_size=1, max_size=3))

    def one(traj):
        t0 = draw(st.sampled_from(anchors))
        return [traj, 0, draw(coord), draw(coord), draw(coord), t0, draw(coord), draw(coord), draw(coord),
                t0 + draw(span_val)]

    rows = [one(k) for k in range(draw(st.integers(1, 6)))]
    cols = [one(100 + k) for k in range(draw(st.integers(1, 6)))]
    return rows, cols


def _store(recs):
    a = np.array(recs, dtype=np.float64)
    return tsk.SegmentStore(a[:, 0].astype(np.int64), a[:, 1].astype(np.int64), *(a[:, k] for k in range(2, 10)))


def _cols(s):
    return {k: getattr(s, k) for k in ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")}


def _hits(rows, cols, d, swap=False):
    h = tsk.pair_intervals(cols, rows, d) if swap else tsk.pair_intervals(rows, cols, d)
    ri, ci = (h.col_idx, h.row_idx) if swap else (h.row_idx, h.col_idx)
    return {(int(r), int(c)): (float(b), float(e)) for r, c, b, e in zip(ri, ci, h.t_begin, h.t_end)}


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if tsk.device_count() < 1:
        pytest.fail("no CUDA device visible for a -m gpu test")
    tsk.set_device(0)


@given(meshes(), dist)
@settings(max_examples=60, deadline=None)
def test_pair_intervals_are_symmetric_and_match_the_oracle(mesh, d):
    rows, cols = (_store(m) for m in mesh)
    fwd = _hits(rows, cols, d)
    assert fwd == _hits(rows, cols, d, swap=True)
    ri, ci, tb, te, _, _ = orc.pair_mesh(_cols(rows), _cols(cols), d)
    assert fwd == {(int(r), int(c)): (float(b), float(e)) for r, c, b, e in zip(ri, ci, tb, te)}


@given(meshes(), dist, dist)
@settings(max_examples=60, deadline=None)
def test_pair_intervals_grow_with_distance(mesh, d1, d2):
    rows, cols = (_store(m) for m in mesh)
    lo, hi = sorted((d1, d2))
    small, big = _hits(rows, cols, lo), _hits(rows, cols, hi)
    for k, (b, e) in small.items():
        assert k in big
        slack = 1e-12 * max(1.0, abs(b), abs(e))
        assert big[k][0] <= b + slack and big[k][1] >= e - slack


@given(meshes(), dist)
@settings(max_examples=60, deadline=None)
def test_pair_intervals_stay_inside_the_shared_span(mesh, d):
    rows, cols = (_store(m) for m in mesh)
    for (r, c), (b, e) in _hits(rows, cols, d).items():
        ta = max(rows.ts[r], cols.ts[c])
        tb = min(rows.te[r], cols.te[c])
        assert ta <= b <= e <= tb
