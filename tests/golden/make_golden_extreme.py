"""Golden vectors for non-finite intermediates, made by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_extreme.py

Pins core.pair_intervals (/root/reference/pkg/src/trajseek/core.py:464-565)
on meshes whose arithmetic overflows: |coordinates| from 1e150 to 1e300,
d up to 1e300.  There aa = |w|^2, cc or the discriminant become inf/NaN,
and the vectorized np.minimum / np.maximum (core.py:545-546) propagate NaN
roots into a miss (core.py:549-553); and on "absorbed offset" pairs, where
cc = |U|^2 loses a perpendicular offset (tests/helpers.py
absorbed_offset_pairs).  Writes extreme.npz next to this file.
"""

from __future__ import annotations

import os
import sys
import warnings

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from trajseek import core  # noqa: E402  (the reference)

from helpers import STORE_FIELDS  # noqa: E402


def store(rows):
    rows = np.asarray(rows, np.float64)
    n = rows.shape[0]
    return {"traj": np.arange(n, dtype=np.int64), "seg": np.zeros(n, np.int64),
            "xs": rows[:, 0], "ys": rows[:, 1], "zs": rows[:, 2], "ts": rows[:, 3],
            "xe": rows[:, 4], "ye": rows[:, 5], "ze": rows[:, 6], "te": rows[:, 7]}


def scenes():
    # 1. head-on from a common start at 1e160 per unit time: aa = inf,
    #    disc = +inf, qq = -inf, r1 = NaN, r2 = 0 -> the reference misses
    yield "headon", store([[0, 0, 0, 0, 1e160, 0, 0, 1]]), store([[0, 0, 0, 0, -1e160, 0, 0, 1]]), 1.0
    yield "headon_d0", store([[0, 0, 0, 0, 1e160, 0, 0, 1]]), store([[0, 0, 0, 0, -1e160, 0, 0, 1]]), 0.0
    # 2. random meshes with mixed magnitudes
    rng = np.random.default_rng(4242)
    for tag, mags, dvals in (("m150", [1e150, 1e153, 1e155, 1.0], [1.0, 1e150, 1e155]),
                             ("m300", [1e300, 1e200, 1e-300, 1.0], [0.0, 2.0, 1e300]),
                             ("mix", [1e160, 1e154, 1e10, 1.0, 0.0], [3.0, 1e154])):
        def rand(n):
            mag = rng.choice(mags, size=(n, 6))
            pos = rng.uniform(-1, 1, (n, 6)) * mag
            still = rng.random(n) < 0.2  # stationary segments
            pos[still, 3:6] = pos[still, 0:3]
            t0 = rng.uniform(0, 4, n)
            span = rng.uniform(0, 2, n)
            span[rng.random(n) < 0.15] = 0.0
            # some segments share a start point with their neighbours
            share = rng.random(n) < 0.3
            pos[share, 0:3] = pos[0, 0:3]
            return np.column_stack([pos[:, 0:3], t0, pos[:, 3:6], t0 + span])
        R, C = rand(16), rand(16)
        for k, d in enumerate(dvals):
            yield f"{tag}_d{k}", store(R), store(C), d
    # 3. absorbed offsets: long motion across the query with a perpendicular
    #    offset h below the rounding of |U|^2: the reference's cc loses h^2
    #    and it reports hits at thresholds far below h (the box cull's radius
    #    needs its box-diagonal term, filter.cuh)
    from helpers import absorbed_offset_pairs

    A, B = absorbed_offset_pairs(24, 777)
    for k, d in enumerate((1e-9, 1e-12, 0.0, 1e-4)):
        yield f"absorbed_d{k}", store(A), store(B), d


def main():
    out = {}
    for tag, r, c, d in scenes():
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            with np.errstate(all="ignore"):
                R = core.SegmentStore(*(r[k] for k in STORE_FIELDS))  # start-time sorted
                C = core.SegmentStore(*(c[k] for k in STORE_FIELDS))
                h = core.pair_intervals(R, C, d)
        for k in STORE_FIELDS:
            out[f"{tag}_rows_{k}"] = np.asarray(getattr(R, k)).copy()
            out[f"{tag}_cols_{k}"] = np.asarray(getattr(C, k)).copy()
        out[f"{tag}_d"] = np.float64(d)
        out[f"{tag}_row_idx"] = h.row_idx
        out[f"{tag}_col_idx"] = h.col_idx
        out[f"{tag}_t_begin"] = h.t_begin
        out[f"{tag}_t_end"] = h.t_end
        out[f"{tag}_misses"] = np.array([h.temporal_misses, h.spatial_misses], np.int64)
        print(tag, "hits", h.row_idx.shape[0], "misses", h.temporal_misses, h.spatial_misses)
    out["tags"] = np.array([t for t, *_ in scenes()])
    path = os.path.join(HERE, "extreme.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
