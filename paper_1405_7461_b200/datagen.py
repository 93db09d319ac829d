"""Synthetic trajectory stores for tests and benchmarks (host side).

RandWalk profiles draw the same PCG64 stream, call for call, as the
reference generator (/root/reference/pkg/src/trajseek/datagen.py:106-267),
so a (profile, seed) pair yields the reference's dataset byte for byte —
that is pinned by tests/golden/datagen.npz.  The data generator itself is
outside the hot path; it exists so the benchmark and the
parity tests feed identical float64 inputs to the GPU path and the CPU
baseline.

``galaxy`` adds the Galaxy-shaped star-orbit workload of the paper
 that the reference does not ship: stars on circular
orbits in a flat rotation curve with small vertical oscillation, sampled
once per time unit.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from .core import DomainError, FormatError, SegmentStore

PROFILE_KINDS = ("uniform", "normal", "normal5", "exp")

CSV_HEADER = ["traj_id", "seg_id", "x_s", "y_s", "z_s", "t_s", "x_e", "y_e", "z_e", "t_e"]


@dataclass(frozen=True)
class GenProfile:
    """Dataset recipe (datagen.py:106-145)."""

    kind: str
    trajectories: int
    seed: int
    timesteps: int = 400
    start_window: tuple[float, float] = (0.0, 100.0)
    normal_mean: float = 200.0
    normal_std: float = 200.0
    exp_mean: float = 70.0
    steps_min: int = 2
    steps_max: int = 1000
    step_scale: float = 1.0
    arena: float = 100.0

    def __post_init__(self) -> None:
        if self.kind not in PROFILE_KINDS:
            raise DomainError(f"unknown profile kind {self.kind!r}; expected one of {PROFILE_KINDS}")
        if self.trajectories < 1:
            raise DomainError(f"trajectories={self.trajectories} must be >= 1")
        if self.timesteps < 2:
            raise DomainError(f"timesteps={self.timesteps} must be >= 2 (one segment)")
        if self.steps_min < 2:
            raise DomainError(f"steps_min={self.steps_min} must be >= 2")
        if self.steps_max < self.steps_min:
            raise DomainError(f"steps_max={self.steps_max} must be >= steps_min")
        lo, hi = self.start_window
        if hi < lo:
            raise DomainError(f"start_window {self.start_window} is inverted")
        if min(self.exp_mean, self.step_scale, self.arena) <= 0:
            raise DomainError("exp_mean, step_scale and arena must be positive")


_DEFAULT_WINDOWS = {"normal": (0.0, 400.0), "normal5": (0.0, 400.0), "exp": (0.0, 20.0)}


def make_profile(kind: str, trajectories: int, seed: int, **overrides) -> GenProfile:
    """Profile with the per-kind default start window (datagen.py:148-159)."""
    p = GenProfile(kind=kind, trajectories=trajectories, seed=seed)
    if kind in _DEFAULT_WINDOWS and "start_window" not in overrides:
        p = replace(p, start_window=_DEFAULT_WINDOWS[kind])
    return replace(p, **overrides) if overrides else p


def _truncated(rng, sampler, lo: float, hi: float, n: int) -> np.ndarray:
    """Rejection-sample n values of ``sampler`` into [lo, hi]."""
    got = []
    need = n
    while need > 0:
        x = sampler(rng, need)
        x = x[(x >= lo) & (x <= hi)]
        got.append(x)
        need -= x.shape[0]
    return np.concatenate(got) if got else np.empty(0)


def _starts(p: GenProfile, rng) -> np.ndarray:
    lo, hi = p.start_window
    n = p.trajectories
    if p.kind in ("uniform", "exp"):
        return rng.uniform(lo, hi, n)
    if p.kind == "normal":
        return _truncated(rng, lambda r, k: r.normal(p.normal_mean, p.normal_std, k), lo, hi, n)
    width = hi - lo
    centres = lo + width * (2 * np.arange(5) + 1) / 10.0
    sd = width / 20.0
    comp = rng.integers(0, 5, n)
    out = np.empty(n, dtype=np.float64)
    for k in range(5):
        sel = comp == k
        if sel.any():
            out[sel] = _truncated(rng, lambda r, m: r.normal(centres[k], sd, m), lo, hi, int(sel.sum()))
    return out


def _lengths(p: GenProfile, rng) -> np.ndarray:
    if p.kind != "exp":
        return np.full(p.trajectories, p.timesteps, dtype=np.int64)
    raw = _truncated(rng, lambda r, k: r.exponential(p.exp_mean, k),
                     float(p.steps_min), float(p.steps_max), p.trajectories)
    return np.rint(raw).astype(np.int64)


def generate(profile: GenProfile) -> SegmentStore:
    """Random-walk store for ``profile`` (datagen.py:206-245), sorted by start."""
    c = generate_columns(profile)
    return SegmentStore(*(c[k] for k in ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")),
                        validate=False)


def generate_columns(profile: GenProfile) -> dict:
    """The unsorted columns of :func:`generate` (trajectory-major order)."""
    rng = np.random.default_rng(profile.seed)
    starts = _starts(profile, rng)
    pts = _lengths(profile, rng)
    nseg = pts - 1
    total = int(nseg.sum())
    cols = {k: np.empty(total, dtype=np.float64) for k in ("xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")}
    traj = np.repeat(np.arange(profile.trajectories, dtype=np.int64), nseg)
    offs = np.concatenate([[0], np.cumsum(nseg)])
    seg = np.arange(total, dtype=np.int64) - np.repeat(offs[:-1], nseg)
    zero = np.zeros((1, 3))
    for i in range(profile.trajectories):
        k = int(nseg[i])
        a, b = int(offs[i]), int(offs[i + 1])
        origin = rng.uniform(0.0, profile.arena, 3)
        walk = origin + np.vstack([zero, np.cumsum(rng.normal(0.0, profile.step_scale, (k, 3)), axis=0)])
        t = starts[i] + np.arange(k + 1, dtype=np.float64)
        cols["ts"][a:b] = t[:-1]
        cols["te"][a:b] = t[1:]
        for ax, (s, e) in enumerate((("xs", "xe"), ("ys", "ye"), ("zs", "ze"))):
            cols[s][a:b] = walk[:-1, ax]
            cols[e][a:b] = walk[1:, ax]
    cols["traj"] = traj
    cols["seg"] = seg
    return cols


def sample_queries(source: SegmentStore, num_traj: int, seed: int) -> SegmentStore:
    """Whole trajectories drawn without replacement (datagen.py:248-267)."""
    ids = np.unique(source.traj)
    if not 1 <= num_traj <= ids.shape[0]:
        raise DomainError(f"num_traj={num_traj} must be in 1..{ids.shape[0]} (distinct trajectories)")
    pick = np.random.default_rng(seed).choice(ids, size=num_traj, replace=False)
    keep = np.isin(source.traj, pick)
    return SegmentStore(*(getattr(source, k)[keep] for k in
                          ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")),
                        validate=False)


def galaxy(stars: int, seed: int, *, points: int = 401, start_window=(0.0, 100.0),
           r_min: float = 1.0, r_max: float = 50.0, v_circ: float = 0.2,
           z_amp: float = 0.5) -> SegmentStore:
    """Galaxy-shaped store: ``stars`` orbits of ``points`` samples each.

    Flat rotation curve (angular speed v_circ / r), uniform disc surface
    density, small vertical epicycles; start times uniform over the
    window (PAPER.md:1025-1031 describes the workload).
    """
    rng = np.random.default_rng(seed)
    r = np.sqrt(rng.uniform(r_min * r_min, r_max * r_max, stars))
    phase = rng.uniform(0.0, 2 * np.pi, stars)
    zphase = rng.uniform(0.0, 2 * np.pi, stars)
    t0 = rng.uniform(start_window[0], start_window[1], stars)
    k = np.arange(points, dtype=np.float64)
    omega = (v_circ / r)[:, None]
    ang = phase[:, None] + omega * k[None, :]
    x = r[:, None] * np.cos(ang)
    y = r[:, None] * np.sin(ang)
    z = z_amp * np.sin(zphase[:, None] + 3.0 * omega * k[None, :])
    t = t0[:, None] + k[None, :]
    traj = np.repeat(np.arange(stars, dtype=np.int64), points - 1)
    seg = np.tile(np.arange(points - 1, dtype=np.int64), stars)
    s, e = (slice(None), slice(None, -1)), (slice(None), slice(1, None))
    return SegmentStore(traj, seg, x[s].ravel(), y[s].ravel(), z[s].ravel(), t[s].ravel(),
                        x[e].ravel(), y[e].ravel(), z[e].ravel(), t[e].ravel(), validate=False)


# ── CSV persistence (datagen.py:273-333), native ─────────────────────────────


def save(store: SegmentStore, path: str) -> None:
    """Write the store as CSV in ordinal order; floats in shortest
    round-trip (repr) form, byte-identical to the reference's save."""
    from . import _native

    _native.save_store_csv(store, path)


def load(path: str, *, strict: bool = False) -> SegmentStore:
    """Read a segment CSV (validation and FormatError messages of
    datagen.py:288-333); rows are sorted by start time unless ``strict``,
    where unsorted input is an error.  Lines the fast native parser cannot
    read (quoted fields, numeric underscores) are re-read by the csv module
    so the accepted syntax matches the reference."""
    from . import _native

    try:
        cols = _native.load_store_csv(path, strict)
    except FormatError as exc:
        # Python-formatted messages (header repr, float() errors) and the
        # rarer syntaxes csv/float() accept come from the csv-module reader
        if "unparsable field" not in str(exc) and "bad header" not in str(exc):
            raise
        cols = _load_python(path, strict)
    return SegmentStore.from_columns(cols, validate=False)


def _load_python(path: str, strict: bool) -> dict:
    import csv

    rows = []
    with open(path, newline="") as fh:
        reader = csv.reader(fh)
        try:
            header = next(reader)
        except StopIteration:
            raise FormatError(f"{path}: empty file") from None
        if header != CSV_HEADER:
            raise FormatError(f"{path}: bad header {header!r}")
        for lineno, row in enumerate(reader, start=2):
            if not row:
                continue
            if len(row) != 10:
                raise FormatError(f"{path}:{lineno}: expected 10 fields, got {len(row)}")
            try:
                vals = (int(row[0]), int(row[1]), *(float(v) for v in row[2:]))
            except ValueError as exc:
                raise FormatError(f"{path}:{lineno}: {exc}") from None
            if not all(np.isfinite(v) for v in vals[2:]):
                raise FormatError(f"{path}:{lineno}: non-finite coordinate")
            if vals[9] < vals[5]:
                raise FormatError(f"{path}:{lineno}: segment ends at t={vals[9]!r} "
                                  f"before it starts at t={vals[5]!r}")
            rows.append(vals)
    if not rows:
        raise FormatError(f"{path}: no segments")
    arr = np.asarray(rows, dtype=np.float64)
    if strict and (np.diff(arr[:, 5]) < 0).any():
        bad = int(np.argmax(np.diff(arr[:, 5]) < 0)) + 3
        raise FormatError(f"{path}:{bad}: rows not sorted by t_s (strict mode)")
    names = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")
    return {k: (arr[:, i].astype(np.int64) if i < 2 else arr[:, i].copy()) for i, k in enumerate(names)}


def write_results(result, path: str, canonical: bool = False) -> None:
    """The search result CSV of the reference CLI (cli.py:62-77), written
    natively; ``canonical`` first applies ResultSet.canonical_order."""
    from . import _native

    if canonical:
        result = result.canonical_order()
    _native.write_results_csv({k: getattr(result, k) for k in
                               ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")},
                              path)
