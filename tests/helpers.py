"""Shared test helpers (no product or oracle logic here)."""

from __future__ import annotations

import hashlib
import os

import numpy as np

STORE_FIELDS = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def random_store_arrays(rng, n, first_traj=0, allow_waypoints=True):
    """Unsorted columns of a random store; draws the same stream as the
    reference test helper (/root/reference/pkg/tests/test_core.py:231-246):
    ~10% waypoints (zero extent) and ~10% stationary segments."""
    t0 = rng.uniform(0.0, 8.0, n)
    span = rng.uniform(0.0, 3.0, n)
    if not allow_waypoints:
        span = np.maximum(span, 1e-3)
    elif n > 0:
        span[rng.random(n) < 0.1] = 0.0
    pos = rng.uniform(-8.0, 8.0, (n, 3))
    step = rng.normal(0.0, 3.0, (n, 3))
    step[rng.random(n) < 0.1] = 0.0
    end = pos + step
    return {
        "traj": np.arange(first_traj, first_traj + n, dtype=np.int64),
        "seg": np.zeros(n, dtype=np.int64),
        "xs": pos[:, 0].copy(), "ys": pos[:, 1].copy(), "zs": pos[:, 2].copy(), "ts": t0,
        "xe": end[:, 0].copy(), "ye": end[:, 1].copy(), "ze": end[:, 2].copy(), "te": t0 + span,
    }


def store_digest(arrays) -> bytes:
    h = hashlib.sha256()
    for k in STORE_FIELDS:
        a = np.ascontiguousarray(arrays[k])
        h.update(k.encode())
        h.update(a.tobytes())
    return h.digest()


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_store(z, prefix):
    return {k: z[f"{prefix}_{k}"] for k in STORE_FIELDS}


def c9_population(n, seed):
    """Pair population of the reference acceptance criterion 9
    (/root/reference/pkg/tests/test_acceptance.py:322-333): the second
    segment starts inside the first's span, ~10% instantaneous segments,
    ~10% stationary first segments.  Returns (A, B) as (n, 8) arrays of
    xs ys zs ts xe ye ze te."""
    rng = np.random.default_rng(seed)
    base = rng.uniform(-50.0, 50.0, n)
    span_a = rng.uniform(0.0, 3.0, n)
    span_a[rng.random(n) < 0.1] = 0.0
    off_b = rng.uniform(-0.5, 0.5, n) * span_a
    span_b = rng.uniform(0.0, 3.0, n)
    span_b[rng.random(n) < 0.1] = 0.0
    coords = rng.uniform(-2.0, 2.0, (n, 12))
    stationary = rng.random(n) < 0.1
    coords[stationary, 3:6] = coords[stationary, 0:3]
    A = np.column_stack([coords[:, 0:3], base, coords[:, 3:6], base + span_a])
    B = np.column_stack([coords[:, 6:9], base + off_b, coords[:, 9:12], base + off_b + span_b])
    return A, B


def absorbed_offset_pairs(n, seed, scale=1000.0):
    """(A, B) as (n, 8) arrays of xs ys zs ts xe ye ze te: pair k moves A_k
    along one axis straight across the stationary (or co-moving) B_k during
    [4k, 4k + 1], offset perpendicular by h = scale * 2^-(18..37).  Below
    h ~ 2^-26 |U| the reference's cc = |U|^2 absorbs h^2, so it reports a
    hit at any threshold d << h (filter.cuh, box cull; tools/filter_check.cpp
    mode 8)."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, 8))
    B = np.zeros((n, 8))
    for k in range(n):
        ax = int(rng.integers(3))
        px = (ax + 1 + int(rng.integers(2))) % 3
        c = rng.uniform(-scale, scale, 3) * (rng.random() < 0.5)
        h = scale * np.ldexp(rng.uniform(0.5, 1.0), -int(18 + rng.integers(20)))
        s, e = c.copy(), c.copy()
        s[ax] += scale * rng.uniform(0.5, 1.0)
        e[ax] -= scale * rng.uniform(0.5, 1.0)
        s[px] += h
        e[px] += h
        qe = c.copy()
        if rng.random() < 0.5:  # the query moves along too (offset kept)
            m = scale * rng.uniform(-1, 1)
            qe[ax] += m
            e[ax] += m
        t0 = 4.0 * k
        A[k] = [*s, t0, *e, t0 + 1.0]
        B[k] = [*c, t0, *qe, t0 + 1.0]
    return A, B
