"""CPU tests of the host side of the drop-in (no GPU needed).

Covers: the C-ABI library loads and exports every symbol include/trajseek.h
declares; the scalar geometry, host candidate-range lookups, planners and
data generator against golden vectors made by the reference; validation
and DomainError behaviour.
"""

from __future__ import annotations

import os
import re

import numpy as np
import pytest

import paper_1405_7461_b200 as tsk
from helpers import GOLDEN, STORE_FIELDS, c9_population, golden_store, load_golden, store_digest
from oracle import oracle as orc
from paper_1405_7461_b200 import _native
from paper_1405_7461_b200.index import TemporalBin, TemporalIndex

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _store(arr):
    return tsk.SegmentStore(*(arr[k] for k in STORE_FIELDS))


def host_index(store, m, rule="member_extents"):
    """A TemporalIndex assembled from the CPU oracle (for CPU-only planner tests)."""
    o = orc.index_build({k: getattr(store, k) for k in STORE_FIELDS}, m, rule)
    bins = [TemporalBin(None, None, None, None)] * m
    occ = np.nonzero(o["nonempty"])[0]
    for k, j in enumerate(occ):
        bins[j] = TemporalBin(float(o["ne_start"][k]), float(o["ne_end"][k]),
                              int(o["ne_first"][k]), int(o["ne_last"][k]))
    return TemporalIndex(m, o["width"], o["t0"], o["t_max"], rule, tuple(bins), o["ne_start"],
                         o["ne_end"], o["ne_first"], o["ne_last"], None, store)


# ── C-ABI surface ───────────────────────────────────────────────────────────


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "trajseek.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t|const char \*)\s*\*?\s*(tsk_\w+)\(",
                              header, flags=re.M))
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    lib = _native.load()
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.tsk_abi_version() == 1


def test_library_is_built_for_sm_100a():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_device_calls_fail_loudly_without_a_gpu():
    if _native.device_count() > 0:
        pytest.skip("a GPU is visible")
    s = tsk.SegmentStore(np.array([0]), np.array([0]), *[np.array([0.0])] * 3, np.array([0.0]),
                         *[np.array([1.0])] * 3, np.array([1.0]))
    with pytest.raises(RuntimeError):
        tsk.build_index(s, 4)
    with pytest.raises(RuntimeError):
        tsk.pair_intervals(s, s, 1.0)


# ── scalar geometry (core.py:309-438) ───────────────────────────────────────


def _seg(v, traj=0):
    return tsk.TrajectorySegment(traj, 0, tsk.SpacetimePoint(*v[0:4]), tsk.SpacetimePoint(*v[4:8]))


def _scalar(a, b, d):
    clip = tsk.temporal_intersection(_seg(a), _seg(b))
    if clip is None:
        return None
    iv = tsk.threshold_interval(clip[0], clip[1], d)
    return None if iv is None else (iv.begin, iv.end)


def test_scalar_geometry_hand_cases():
    z = load_golden("pairs.npz")
    for a, b, d, want in zip(z["hand_a"], z["hand_b"], z["hand_d"], z["hand_res"]):
        expect = None if want[0] == 0.0 else (want[1], want[2])
        assert _scalar(tuple(a), tuple(b), float(d)) == expect


def test_scalar_geometry_c9_population():
    z = load_golden("scalar_c9.npz")
    A, B = c9_population(20_000, 77)
    for i in range(0, A.shape[0], 5):
        want = None if z["res"][i, 0] != 1.0 else (z["res"][i, 1], z["res"][i, 2])
        assert _scalar(tuple(A[i]), tuple(B[i]), 1.0) == want


def test_scalar_validation():
    q = _seg((0, 0, 0, 0, 0, 0, 0, 1))
    e = _seg((0, 0, 0, 0, 0, 0, 0, 2))
    with pytest.raises(tsk.DomainError):
        tsk.threshold_interval(q, e, 1.0)
    for bad in (-1.0, float("nan"), float("inf")):
        with pytest.raises(tsk.DomainError):
            tsk.threshold_interval(q, q, bad)
    with pytest.raises(tsk.DomainError):
        _seg((0, 0, 0, 2, 0, 0, 0, 1))
    with pytest.raises(tsk.DomainError):
        tsk.TimeInterval(2.0, 1.0)
    with pytest.raises(tsk.DomainError):
        tsk.position_at(q, 2.0)
    assert tsk.position_at(q, 0.5) == (0.0, 0.0, 0.0)


# ── store / result containers ───────────────────────────────────────────────


def test_store_sorts_stably_and_validates():
    s = tsk.SegmentStore(np.array([1, 2, 3]), np.zeros(3, np.int64), np.zeros(3), np.zeros(3),
                         np.zeros(3), np.array([5.0, 1.0, 5.0]), np.ones(3), np.zeros(3),
                         np.zeros(3), np.array([6.0, 2.0, 6.0]))
    assert list(s.ts) == [1.0, 5.0, 5.0] and list(s.traj) == [2, 1, 3]
    one = lambda v: np.array([v], dtype=np.float64)  # noqa: E731
    with pytest.raises(tsk.DomainError):
        tsk.SegmentStore(np.array([0]), np.array([0]), one(0), one(0), one(0), one(2.0), one(1),
                         one(0), one(0), one(1.0))
    with pytest.raises(tsk.DomainError):
        tsk.SegmentStore(np.array([0]), np.array([0]), one(np.nan), one(0), one(0), one(0.0),
                         one(1), one(0), one(0), one(1.0))
    with pytest.raises(AttributeError):
        s.ts = None
    v = s.view(1, 2)
    assert len(v) == 2 and v.segment(0) == s.segment(1)
    assert s.range_extent(0, 2) == tsk.TimeInterval(1.0, 6.0)
    with pytest.raises(tsk.DomainError):
        s.view(2, 5)


def test_store_matches_oracle_order_on_random_input():
    z = load_golden("pairs.npz")
    rng = np.random.default_rng(1234)
    from helpers import random_store_arrays

    s = _store(random_store_arrays(rng, 40))
    for k in STORE_FIELDS:
        assert np.array_equal(getattr(s, k), z[f"s1234_rows_{k}"])


def test_result_set_canonical_order():
    a = tsk.ResultSet(np.array([2, 1]), np.array([0, 0]), np.array([7, 9]), np.array([1, 0]),
                      np.array([0.5, 0.25]), np.array([1.0, 0.75]))
    merged = tsk.ResultSet.concatenate([a, tsk.ResultSet.empty()])
    o = merged.canonical_order()
    assert list(o.query_traj) == [1, 2]
    items = list(o.items())
    assert items[0].entry_traj_id == 9 and items[0].interval == tsk.TimeInterval(0.25, 0.75)
    assert o.key_array().shape == (2, 6)


# ── candidate ranges (index.py:149-173) on the host ─────────────────────────


def test_host_candidate_ranges_match_golden():
    z = load_golden("index.npz")
    tags = sorted({k.split("_")[0] for k in z.files if k.endswith("_qb")})
    checked = 0
    for tag in tags:
        st = _store(golden_store(z, tag))
        ms = sorted({int(k.split("_")[1][1:]) for k in z.files
                     if k.startswith(tag + "_m") and k.endswith("_hdr")})
        for m in ms:
            for rule in ("member_extents", "grid_start"):
                key = f"{tag}_m{m}_{rule}"
                ix = host_index(st, m, rule)
                want = z[f"{key}_ranges"]
                f, l = tsk.candidate_ranges(ix, z[f"{tag}_qb"], z[f"{tag}_qe"])
                assert np.array_equal(np.column_stack([f, l]), want), key
                for (b, e), w in zip(zip(z[f"{tag}_qb"], z[f"{tag}_qe"]), want):
                    got = tsk.candidate_range(ix, tsk.TimeInterval(float(b), float(e)))
                    assert got == (None if w[0] < 0 else tuple(w))
                checked += 1
    assert checked >= 20


def test_four_bin_fixture_counts():
    """Figure-1/2 stores of the reference fixtures (tests/fixtures.py:66-158)."""
    ext = [(0.0, 1.7), (0.6, 1.5), (0.7, 1.3), (1.9, 3.7), (2.5, 7.5), (2.8, 4.6), (3.9, 5.5),
           (4.1, 5.8), (4.8, 6.2), (6.5, 9.4), (7.0, 7.8), (8.3, 11.0), (9.3, 11.5),
           (10.4, 12.0), (11.6, 11.9)]
    st = _extents_store(ext)
    ix = host_index(st, 4)
    assert tuple((b.first, b.last) for b in ix.bins) == ((0, 5), (6, 8), (9, 11), (12, 14))
    assert tuple(b.end for b in ix.bins) == (7.5, 6.2, 11.0, 12.0)
    groups = [(0.1, 5.2), (4.8, 6.1), (5.7, 9.1), (8.0, 9.2), (8.5, 10.5), (11.5, 12.0)]
    qext, qtraj = [], []
    for g, (b, e) in enumerate(groups):
        for k in range(9):
            qext.append((b + k * 1e-3, b + k * 1e-3 + 1e-3))
            qtraj.append(g)
        qext.append((b + 9e-3, e))
        qtraj.append(g)
    q = _extents_store(qext, qtraj)
    plan = tsk.periodic(q, 10, ix)
    assert [b.interactions for b in plan.batches] == [90, 90, 120, 30, 60, 30]
    assert tsk.count_interactions_naive(ix, plan) == [90, 90, 120, 30, 60, 30]
    assert tsk.periodic(q, 60, ix).total_interactions == 900
    gix = host_index(st, 4, "grid_start")
    assert [b.interactions for b in tsk.periodic(q, 10, gix).batches] == [90, 120, 150, 60, 60, 30]


def _extents_store(ext, traj=None):
    n = len(ext)
    ts = np.array([a for a, _ in ext])
    te = np.array([b for _, b in ext])
    xs = np.arange(n, dtype=np.float64)
    z = np.zeros(n)
    return tsk.SegmentStore(np.arange(n) if traj is None else np.array(traj), z.astype(np.int64),
                            xs, z, z, ts, xs + 1.0, z, z, te)


# ── planners (planner.py:202-429) ───────────────────────────────────────────


def _table(plan):
    return np.array([(b.lo, b.hi, -1 if b.first is None else b.first,
                      -1 if b.last is None else b.last) for b in plan.batches], dtype=np.int64)


@pytest.mark.parametrize("tag", ["p41", "p47", "p59", "p57"])
def test_planners_match_reference_golden(tag):
    z = load_golden("plans.npz")
    e = _store(golden_store(z, f"{tag}_e"))
    q = _store(golden_store(z, f"{tag}_q"))
    ix = host_index(e, int(z[f"{tag}_m"]))
    plans = {
        "periodic7": tsk.periodic(q, 7, ix), "periodic25": tsk.periodic(q, 25, ix),
        "fixed1": tsk.setsplit_fixed(q, ix, 1), "fixed9": tsk.setsplit_fixed(q, ix, 9),
        "fixed17": tsk.setsplit_fixed(q, ix, 17),
        "minmax3_10": tsk.setsplit_minmax(q, ix, 3, 10), "minmax5_18": tsk.setsplit_minmax(q, ix, 5, 18),
        "max6": tsk.setsplit_max(q, ix, 6), "max11": tsk.setsplit_max(q, ix, 11),
        "gmin4": tsk.greedy_min(q, ix, 4), "gmin8": tsk.greedy_min(q, ix, 8),
        "gmax4": tsk.greedy_max(q, ix, 4), "gmax8": tsk.greedy_max(q, ix, 8),
    }
    for name, p in plans.items():
        assert np.array_equal(_table(p), z[f"{tag}_{name}"]), name
    for k in (1, 5, 17):
        assert tsk.setsplit_fixed(q, ix, k).sizes() == tsk.setsplit_fixed(q, ix, k, literal=True).sizes()
    assert tsk.setsplit_minmax(q, ix, 5, 18).sizes() == \
        tsk.setsplit_minmax(q, ix, 5, 18, literal=True).sizes()


def test_greedy_ladder_and_validation():
    entries = _extents_store([(float(i), i + 0.5) for i in range(10)])
    ix = host_index(entries, 10)
    q = _extents_store([(i + 0.1, i + 0.2) for i in range(10)], range(50, 60))
    assert tsk.greedy_min(q, ix, 3).sizes() == [3, 3, 3, 1]
    assert tsk.greedy_max(q, ix, 3).sizes() == [4, 4, 2]
    for bad in (lambda: tsk.greedy_min(q, ix, 0), lambda: tsk.greedy_max(q, ix, -2),
                lambda: tsk.setsplit_fixed(q, ix, 0), lambda: tsk.setsplit_minmax(q, ix, 10, 5),
                lambda: tsk.periodic(q, 0, ix)):
        with pytest.raises(tsk.DomainError):
            bad()
    good = tsk.periodic(q, 5, ix)
    a, b = good.batches
    with pytest.raises(tsk.DomainError):
        tsk.BatchPlan(q, (a, tsk.QueryBatch(b.lo + 1, b.hi, b.extent, b.first, b.last)))
    with pytest.raises(tsk.DomainError):
        tsk.BatchPlan(q, ())


def test_engine_validates_before_touching_the_device():
    s = _extents_store([(0.0, 1.0), (0.5, 2.0)])
    q = _extents_store([(0.0, 1.0)])
    with pytest.raises(tsk.DomainError):
        tsk.execute_batch(s, q, (0, 5), 1.0)
    with pytest.raises(tsk.DomainError):
        tsk.execute_batch(s, q, (0, 1), 1.0, workers=0)
    with pytest.raises(tsk.DomainError):
        tsk.resolve_workers(0)
    assert tsk.resolve_workers(3) == 3


# ── data generator (datagen.py:106-267) ─────────────────────────────────────


def test_datagen_reproduces_reference_streams():
    z = load_golden("datagen.npz")
    cases = [("uniform", 5, 3, {}), ("normal", 7, 4, {}), ("normal5", 9, 5, {}),
             ("exp", 30, 6, {}), ("uniform", 3, 7, {"timesteps": 20, "step_scale": 2.5})]
    for i, (kind, n, seed, kw) in enumerate(cases):
        s = tsk.generate(tsk.make_profile(kind, n, seed=seed, **kw))
        arr = {k: getattr(s, k) for k in STORE_FIELDS}
        assert store_digest(arr) == z[f"g{i}"].tobytes(), kind
        assert len(s) == int(z[f"g{i}_n"])
        q = tsk.sample_queries(s, max(1, n // 2), seed=seed + 100)
        assert store_digest({k: getattr(q, k) for k in STORE_FIELDS}) == z[f"g{i}_q"].tobytes()


def test_config1_inputs_match_reference_digest():
    z = load_golden("search.npz")
    store = tsk.generate(tsk.make_profile("uniform", 1000, seed=1, timesteps=100))
    pool = tsk.generate(tsk.make_profile("uniform", 1000, seed=2, timesteps=100))
    q = tsk.sample_queries(pool, 100, seed=3)
    assert store_digest({k: getattr(store, k) for k in STORE_FIELDS}) == z["c1_e_digest"].tobytes()
    assert store_digest({k: getattr(q, k) for k in STORE_FIELDS}) == z["c1_q_digest"].tobytes()


def test_galaxy_shape():
    g = tsk.galaxy(50, seed=1, points=41)
    assert len(g) == 50 * 40
    assert np.all(np.diff(g.ts) >= 0)
    assert np.allclose(g.te - g.ts, 1.0)


# ── native planners (csrc/planner.cu) vs the Python implementations ─────────


@pytest.mark.parametrize("seed", [41, 47, 59, 61])
def test_native_planners_equal_python_planners(seed):
    from helpers import random_store_arrays

    rng = np.random.default_rng(seed)
    e = _store(random_store_arrays(rng, 400))
    q = _store(random_store_arrays(rng, 150, first_traj=10_000))
    ix = host_index(e, 24)
    pairs = [
        (tsk.setsplit_fixed(q, ix, 13), tsk.setsplit_fixed(q, ix, 13, literal=True)),
        (tsk.setsplit_minmax(q, ix, 4, 17), tsk.setsplit_minmax(q, ix, 4, 17, literal=True)),
        (tsk.setsplit_max(q, ix, 9), tsk.setsplit_max(q, ix, 9, literal=True)),
        (tsk.greedy_min(q, ix, 7), tsk.greedy_min(q, ix, 7, native=False)),
        (tsk.greedy_max(q, ix, 7), tsk.greedy_max(q, ix, 7, native=False)),
    ]
    for a, b in pairs:
        assert a.batches == b.batches


def test_native_planners_on_generated_exp_profile():
    store = tsk.generate(tsk.make_profile("exp", 200, seed=71))
    pool = tsk.generate(tsk.make_profile("exp", 100, seed=72))
    q = tsk.sample_queries(pool, 30, seed=73)
    ix = host_index(store, 1000)
    from paper_1405_7461_b200 import planner as P

    R = P._Runs(q, ix)
    P._cheapest_heap(R, None, 120)
    assert tsk.setsplit_max(q, ix, 120).batches == R.plan().batches
    assert tsk.greedy_max(q, ix, 120).batches == tsk.greedy_max(q, ix, 120, native=False).batches
    assert tsk.greedy_min(q, ix, 120).batches == tsk.greedy_min(q, ix, 120, native=False).batches


def test_drop_in_namespace_covers_reference_all():
    """Every name the reference exports (trajseek.__all__, committed from
    /root/reference/pkg/src/trajseek/__init__.py:60-114) is importable from
    the drop-in package and listed in its __all__."""
    import json

    import paper_1405_7461_b200 as tsk

    names = json.load(open(os.path.join(GOLDEN, "reference_all.json")))
    missing = [n for n in names if not hasattr(tsk, n)]
    assert not missing, missing
    assert set(names) <= set(tsk.__all__)


def test_per_batch_behaves_as_a_list():
    """SearchStats.per_batch fills itself before every list operation."""
    from paper_1405_7461_b200.engine import BatchTrace, _LazyTraces

    src = ([3, 4], [10, 0], [30, 0], [2, 0], [0.5, 0.0])
    want = [BatchTrace(0, 3, 10, 30, 2, 0.5), BatchTrace(1, 4, 0, 0, 0, 0.0)]

    def mk():
        return _LazyTraces(src=tuple(list(x) for x in src))

    assert mk().copy() == want
    assert mk() + [] == want and [] + mk() == want
    a = mk()
    a += [want[0]]
    assert a == want + [want[0]]
    b = mk()
    b.clear()
    assert len(b) == 0 and b == []
    assert mk().index(want[1]) == 1 and mk().count(want[0]) == 1
    c = mk()
    c.sort(key=lambda t: -t.ordinal)
    assert c == want[::-1]
    assert mk().pop() == want[1]
    d = mk()
    d[0] = want[1]
    assert d == [want[1], want[1]]
    assert list(mk()) == want and len(mk()) == 2 and mk()[1] == want[1]
    import pickle

    assert pickle.loads(pickle.dumps(mk())) == want


@pytest.mark.parametrize("mode", [0, 1, 4, 8])
def test_plan_units_partition_every_batch_candidate_pair(mode):
    """The work units K1 runs (pairs, staircase quads and octets,
    tsk_internal.cuh) partition the plan: every (batch, candidate) pair of
    every batch's span lies in exactly one unit, a unit's batches are
    consecutive and adjacent in the query order, and its tile offsets are
    the running sums of their sizes.  Random plans with monotone and
    non-monotone spans, empty spans and groups larger than a tile."""
    rng = np.random.default_rng(100 + mode)
    lib = _native.load()
    widest = 0  # most batches in one unit (the staircase must be exercised)
    for trial in range(60):
        nb = int(rng.integers(1, 70))
        sizes = rng.integers(1, 200, nb)
        hi = np.cumsum(sizes) - 1
        lo = hi - sizes + 1
        f = np.cumsum(rng.integers(0, 50, nb))
        if trial % 3 == 0:  # break monotonicity
            f = rng.permutation(f)
        last = f + rng.integers(0, 400, nb)
        if trial % 3 != 0:  # both ends non-decreasing: groups form staircases
            last = np.maximum.accumulate(last)
        empty = rng.random(nb) < (0.1 if trial % 2 else 0.0)
        first = np.where(empty, -1, f).astype(np.int64)
        last = np.where(empty, -1, last).astype(np.int64)
        tqs = int(rng.choice([256, 512, 1024]))
        cap = 16 * nb + 16
        out = np.zeros(13 * cap, np.int64)
        arr = [np.ascontiguousarray(a, dtype=np.int64) for a in (lo, hi, first, last)]
        nu = lib.tsk_plan_units(nb, *[a.ctypes.data_as(_native._PI64) for a in arr], mode, tqs,
                                out.ctypes.data_as(_native._PI64), cap)
        assert nu > 0
        cover = [[] for _ in range(nb)]
        for u in out[:13 * nu].reshape(nu, 13):
            b, b1, lo_q, s, js, jx, uf, ul = u[0], u[1], u[2], u[3], u[4], u[5:11], u[11], u[12]
            if uf > ul:
                continue  # an empty unit holds no work items
            k = 1 if b1 < 0 else 2 + int((jx < s).sum())
            widest = max(widest, k)
            assert b1 < 0 or b1 == b + 1
            assert lo_q == lo[b] and s == sizes[b:b + k].sum()
            offs = np.concatenate([[0], np.cumsum(sizes[b:b + k])[:-1]])
            if k > 1:
                assert js == offs[1] and list(jx[:k - 2]) == list(offs[2:k])
                assert all(lo[g + 1] == hi[g] + 1 for g in range(b, b + k - 1))
            for g in range(b, b + k):
                cover[g].append((int(uf), int(ul)))
        for g in range(nb):
            iv = sorted(cover[g])
            if first[g] < 0:
                assert iv == [], (g, iv)
                continue
            assert iv, g
            assert iv[0][0] == first[g] and iv[-1][1] == last[g], (g, iv, first[g], last[g])
            for (a0, a1), (b0, b1_) in zip(iv, iv[1:]):
                assert b0 == a1 + 1, (g, iv)  # contiguous, no overlap
    assert widest == {0: 1, 1: 2, 4: 4, 8: 8}[mode], widest
