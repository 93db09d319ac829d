"""The reference's own engine/oracle/acceptance tests, run against the GPU path.

Ports of /root/reference/pkg/tests/test_engine.py:23-131,
test_oracle.py:26-124 and test_acceptance.py (criteria 1, 9 and 10) with
the same scenes and assertions, so the drop-in is held to the reference's
contract.  Scenes are rebuilt with the package's datagen (which reproduces
the reference's streams, tests/test_host.py::test_datagen_*).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1405_7461_b200 as tsk
from helpers import c9_population, load_golden, random_store_arrays
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

FIELDS = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")


def _store(arr):
    return tsk.SegmentStore(*(arr[k] for k in FIELDS))


def random_store(rng, n, first_traj=0):
    return _store(random_store_arrays(rng, n, first_traj))


def store_from_extents(extents, traj_ids=None):
    n = len(extents)
    ts = np.array([a for a, _ in extents], dtype=np.float64)
    te = np.array([b for _, b in extents], dtype=np.float64)
    xs = np.arange(n, dtype=np.float64)
    z = np.zeros(n)
    ids = np.arange(n) if traj_ids is None else np.asarray(list(traj_ids))
    return tsk.SegmentStore(ids, z.astype(np.int64), xs, z, z, ts, xs + 1.0, z, z, te)


def seg(traj, x0, y0, z0, t0, x1, y1, z1, t1):
    return tsk.TrajectorySegment(traj, 0, tsk.SpacetimePoint(x0, y0, z0, t0),
                                 tsk.SpacetimePoint(x1, y1, z1, t1))


@pytest.fixture(scope="module")
def small_scene():
    """tests/conftest.py:38-49 of the reference."""
    store = tsk.generate(tsk.make_profile("uniform", 6, seed=3, timesteps=150))
    index = tsk.build_index(store, 60)
    pool = tsk.generate(tsk.make_profile("uniform", 6, seed=8, timesteps=150))
    queries = tsk.sample_queries(pool, 2, seed=11)
    return store, index, queries, 20.0


# ── test_engine.py ──────────────────────────────────────────────────────────


def test_all_hit_batch_saturates_the_counters():
    entries = store_from_extents([(0.0, 4.0)] * 5)
    queries = store_from_extents([(0.0, 4.0)] * 3, traj_ids=(100, 101, 102))
    res, stats = tsk.execute_batch(entries, queries, (0, 4), 1000.0, workers=1)
    assert stats.interactions_computed == 15
    assert stats.hits == len(res) == 15
    assert stats.temporal_misses == stats.spatial_misses == 0
    assert all(item.interval.length > 0 for item in res.items())


def test_disjoint_batch_counts_only_temporal_misses():
    entries = store_from_extents([(0.0, 1.0), (0.5, 2.0)])
    queries = store_from_extents([(5.0, 6.0)], traj_ids=(9,))
    res, stats = tsk.execute_batch(entries, queries, (0, 1), 10.0, workers=1)
    assert len(res) == 0
    assert stats.temporal_misses == 2
    assert stats.spatial_misses == 0


def test_stats_partition_the_interaction_count(small_scene):
    store, index, queries, d = small_scene
    _, stats = tsk.run_search(store, index, tsk.periodic(queries, 40, index), d, workers=1)
    assert stats.interactions_computed > 0
    assert stats.hits + stats.temporal_misses + stats.spatial_misses == stats.interactions_computed
    assert sum(t.interactions for t in stats.per_batch) == stats.interactions_computed
    assert sum(t.hits for t in stats.per_batch) == stats.hits
    assert 0.0 <= stats.wasteful_fraction() <= 1.0
    assert stats.kernel_seconds >= 0.0
    assert stats.total_seconds >= stats.kernel_seconds


def test_run_search_matches_brute_force(small_scene):
    store, index, queries, d = small_scene
    want = tsk.brute_force_search(store, queries, d).canonical_order()
    assert len(want) > 0
    for plan in (tsk.periodic(queries, 25, index), tsk.periodic(queries, len(queries), index),
                 tsk.greedy_min(queries, index, 30), tsk.setsplit_max(queries, index, 40)):
        got, _ = tsk.run_search(store, index, plan, d, workers=1)
        assert np.array_equal(got.canonical_order().key_array(), want.key_array())


def test_worker_count_never_changes_results(small_scene):
    store, index, queries, d = small_scene
    plan = tsk.periodic(queries, 30, index)
    base, base_stats = tsk.run_search(store, index, plan, d, workers=1)
    for workers in (2, 3, 5):
        res, stats = tsk.run_search(store, index, plan, d, workers=workers)
        assert np.array_equal(res.key_array(), base.key_array())
        assert stats.interactions_computed == base_stats.interactions_computed
        assert stats.hits == base_stats.hits
        assert [t.interactions for t in stats.per_batch] == [t.interactions for t in base_stats.per_batch]


def test_result_order_is_deterministic_without_sorting(small_scene):
    store, index, queries, d = small_scene
    plan = tsk.periodic(queries, 17, index)
    a, _ = tsk.run_search(store, index, plan, d, workers=1)
    b, _ = tsk.run_search(store, index, plan, d, workers=4)
    for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end"):
        assert np.array_equal(getattr(a, k), getattr(b, k))


def test_batches_beyond_the_store_are_skipped():
    entries = store_from_extents([(0.0, 1.0), (0.8, 2.0)])
    index = tsk.build_index(entries, 2)
    queries = store_from_extents([(0.5, 1.5), (10.0, 11.0)], traj_ids=(7, 8))
    plan = tsk.periodic(queries, 1, index)
    assert plan.batches[1].first is None
    res, stats = tsk.run_search(entries, index, plan, 100.0, workers=1)
    assert stats.per_batch[1].interactions == 0
    assert set(res.query_traj) == {7}


def test_conservative_candidates_show_up_as_temporal_misses():
    rng = np.random.default_rng(5)
    store = random_store(rng, 50)
    index = tsk.build_index(store, 1)
    queries = store_from_extents([(0.0, 0.2)], traj_ids=(900,))
    want = tsk.brute_force_search(store, queries, 3.0).canonical_order()
    got, stats = tsk.run_search(store, index, tsk.periodic(queries, 1, index), 3.0, workers=1)
    assert stats.interactions_computed == 50
    assert stats.temporal_misses > 0
    assert np.array_equal(got.canonical_order().key_array(), want.key_array())


def test_launch_overhead_pass_is_fast_and_positive(small_scene):
    store, _, queries, _ = small_scene
    t = tsk.launch_overhead_pass(store, queries.view(0, 9), (0, len(store) - 1), workers=1)
    assert 0.0 <= t < 1.0


# ── test_oracle.py (brute force) ────────────────────────────────────────────


def store_of(segments):
    return tsk.SegmentStore.from_segments(list(segments))


def test_hand_scene_single_window():
    entries = store_of([seg(0, 10, 0, 0, 0.0, -10, 0, 0, 1.0)])
    queries = store_of([seg(7, 0, 0, 0, 0.0, 0, 0, 0, 1.0)])
    r = tsk.brute_force_search(entries, queries, 1.0)
    assert len(r) == 1
    assert (r.query_traj[0], r.query_seg[0], r.entry_traj[0], r.entry_seg[0]) == (7, 0, 0, 0)
    assert r.t_begin[0] == pytest.approx(0.45, abs=1e-12)
    assert r.t_end[0] == pytest.approx(0.55, abs=1e-12)


def test_disjoint_and_far_apart_produce_nothing():
    e = store_of([seg(0, 0, 0, 0, 0.0, 0, 0, 0, 1.0)])
    assert len(tsk.brute_force_search(e, store_of([seg(1, 0, 0, 0, 2.0, 0, 0, 0, 3.0)]), 100.0)) == 0
    assert len(tsk.brute_force_search(e, store_of([seg(1, 500, 0, 0, 0.0, 500, 0, 0, 1.0)]), 1.0)) == 0


def test_every_overlapping_pair_hits_at_large_d():
    rng = np.random.default_rng(61)
    entries = random_store(rng, 40)
    queries = random_store(rng, 25, first_traj=900)
    results = tsk.brute_force_search(entries, queries, 1e9)
    overlapping = sum(1 for qi in range(len(queries)) for ei in range(len(entries))
                      if queries.ts[qi] <= entries.te[ei] and entries.ts[ei] <= queries.te[qi])
    assert len(results) == overlapping


def test_query_major_output_order():
    rng = np.random.default_rng(62)
    entries = random_store(rng, 120)
    queries = random_store(rng, 30, first_traj=900)
    results = tsk.brute_force_search(entries, queries, 6.0)
    assert len(results) > 0
    keys = results.key_array()
    order = np.lexsort((keys[:, 3], keys[:, 2], keys[:, 1], keys[:, 0]))
    assert np.array_equal(order, np.arange(len(results)))
    # query-major as emitted: query ordinals (traj ids are unique here) ascend
    qpos = {int(t): i for i, t in enumerate(queries.traj)}
    qo = np.array([qpos[int(t)] for t in results.query_traj])
    assert np.all(np.diff(qo) >= 0)


def test_insertion_order_of_entries_does_not_change_hits():
    rng = np.random.default_rng(64)
    entries = random_store(rng, 80)
    queries = random_store(rng, 20, first_traj=900)
    shuffled = rng.permutation(len(entries))
    reordered = store_of([entries.segment(int(i)) for i in shuffled])
    a = tsk.brute_force_search(entries, queries, 7.0).canonical_order()
    b = tsk.brute_force_search(reordered, queries, 7.0).canonical_order()
    assert np.array_equal(a.key_array(), b.key_array())
    assert np.array_equal(a.t_begin, b.t_begin) and np.array_equal(a.t_end, b.t_end)


def test_brute_force_matches_c_oracle_on_waypoint_heavy_scene():
    from oracle import c_oracle

    rng = np.random.default_rng(65)
    entries = random_store(rng, 3000)
    queries = random_store(rng, 700, first_traj=10**5)
    got = tsk.brute_force_search(entries, queries, 2.0)
    want, _, _ = c_oracle.brute_force({k: getattr(entries, k) for k in FIELDS},
                                      {k: getattr(queries, k) for k in FIELDS}, 2.0)
    for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end"):
        assert np.array_equal(getattr(got, k), want[k]), k


# ── test_acceptance.py ──────────────────────────────────────────────────────


D = 15.0


def _queries(kind, trajectories, seed, sample, sample_seed):
    pool = tsk.generate(tsk.make_profile(kind, trajectories, seed=seed))
    return tsk.sample_queries(pool, sample, seed=sample_seed)


def test_criterion_01_every_planner_matches_brute_force():
    """C1: 3 scenes (>= 20k entries, >= 1k queries) x 8 plans; here bit-exact."""
    scenes = {
        "uniform": (tsk.generate(tsk.make_profile("uniform", 52, seed=11)), _queries("uniform", 10, 21, 3, 31)),
        "normal": (tsk.generate(tsk.make_profile("normal", 52, seed=12)), _queries("normal", 10, 22, 3, 32)),
        "exp": (tsk.generate(tsk.make_profile("exp", 330, seed=13)), _queries("exp", 60, 23, 20, 33)),
    }
    for name, (store, queries) in scenes.items():
        assert len(store) >= 20_000 and len(queries) >= 1_000, name
        index = tsk.build_index(store, 1000)
        want = tsk.brute_force_search(store, queries, D).key_array()
        assert want.shape[0] > 0
        n = len(queries)
        plans = {
            "periodic(64)": tsk.periodic(queries, 64, index),
            "periodic(100)": tsk.periodic(queries, 100, index),
            "periodic(128)": tsk.periodic(queries, 128, index),
            "setsplit_fixed": tsk.setsplit_fixed(queries, index, max(1, math.ceil(n / 100))),
            "setsplit_max": tsk.setsplit_max(queries, index, 100),
            "setsplit_minmax": tsk.setsplit_minmax(queries, index, 16, 100),
            "greedy_min": tsk.greedy_min(queries, index, 100),
            "greedy_max": tsk.greedy_max(queries, index, 100),
        }
        for label, plan in plans.items():
            got, _ = tsk.run_search(store, index, plan, D, workers=1)
            assert np.array_equal(got.key_array(), want), (name, label)


def test_criterion_09_c9_population_on_device():
    """C9 pair population: GPU mesh diagonal equals the reference's scalar
    solver bit for bit on 20k pairs (golden from the reference)."""
    z = load_golden("scalar_c9.npz")
    A, B = c9_population(20_000, 77)
    n = A.shape[0]
    # each pair in its own 1x1 mesh would be 20k launches; instead shift pair i
    # by a multiple of 1024 time units?  That changes rounding — so evaluate the
    # pairs in chunks of 2,000 as meshes and read the diagonal.
    for lo in range(0, n, 2000):
        hi = min(lo + 2000, n)
        k = hi - lo
        rows = tsk.SegmentStore(np.arange(k), np.zeros(k, np.int64), *[A[lo:hi, c] for c in range(8)])
        cols = tsk.SegmentStore(np.arange(k) + 10**6, np.zeros(k, np.int64), *[B[lo:hi, c] for c in range(8)])
        h = tsk.pair_intervals(rows, cols, 1.0)
        got = {}
        rt = rows.traj[h.row_idx]
        ct = cols.traj[h.col_idx] - 10**6
        for a, c, b, e in zip(rt, ct, h.t_begin, h.t_end):
            if a == c:
                got[int(a)] = (b, e)
        for i in range(k):
            res = z["res"][lo + i]
            want = None if res[0] != 1.0 else (res[1], res[2])
            assert got.get(i) == want, lo + i


def test_criterion_10_runs_are_deterministic():
    store = tsk.generate(tsk.make_profile("uniform", 12, seed=5))
    index = tsk.build_index(store, 64)
    queries = _queries("uniform", 8, 6, 2, 7)
    plan = tsk.greedy_max(queries, index, 50)
    outs = [tsk.run_search(store, index, plan, 20.0, workers=w)[0] for w in (1, 1, 3)]
    for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end"):
        assert np.array_equal(getattr(outs[0], k), getattr(outs[1], k))
        assert np.array_equal(getattr(outs[0], k), getattr(outs[2], k))
    assert len(outs[0]) > 1
    # and the engine order equals the reference engine's (oracle port)
    e = {k: getattr(store, k) for k in FIELDS}
    q = {k: getattr(queries, k) for k in FIELDS}
    want, _ = orc.search(e, orc.index_build(e, 64), q,
                         [(b.lo, b.hi, None, None, None, None) for b in plan.batches], 20.0)
    for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end"):
        assert np.array_equal(getattr(outs[0], k), want[k]), k
