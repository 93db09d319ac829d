"""Pin the CPU oracle (oracle/) to golden vectors made by the reference itself.

The golden files come from tests/golden/make_golden.py, which runs the
reference package (/root/reference/pkg/src/trajseek) in the build
container.  These are CPU-only tests.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from helpers import STORE_FIELDS, c9_population, golden_store, load_golden, random_store_arrays
from oracle import c_oracle
from oracle import oracle as orc


def _ostore(arr):
    return orc.make_store(*(arr[k] for k in STORE_FIELDS))


# ── pairs (core.py:464-565) ────────────────────────────────────────────────


def test_hand_cases_numpy_scalar_and_c():
    z = load_golden("pairs.npz")
    for a, b, d, want in zip(z["hand_a"], z["hand_b"], z["hand_d"], z["hand_res"]):
        got_py = orc.pair_scalar(tuple(a), tuple(b), float(d))
        got_c = c_oracle.pair(tuple(a), tuple(b), float(d))
        expect = None if want[0] == 0.0 else (want[1], want[2])
        assert got_py == expect
        assert got_c == expect


@pytest.mark.parametrize("tag", ["s1234", "s99", "s7", "s8"])
def test_pair_mesh_matches_golden_bit_for_bit(tag):
    z = load_golden("pairs.npz")
    rows = golden_store(z, f"{tag}_rows")
    cols = golden_store(z, f"{tag}_cols")
    ri, ci, tb, te, tm, sm = orc.pair_mesh(rows, cols, float(z[f"{tag}_d"]))
    assert np.array_equal(ri, z[f"{tag}_row_idx"])
    assert np.array_equal(ci, z[f"{tag}_col_idx"])
    assert np.array_equal(tb, z[f"{tag}_t_begin"])
    assert np.array_equal(te, z[f"{tag}_t_end"])
    assert [tm, sm] == list(z[f"{tag}_misses"])
    assert tm + sm + ri.shape[0] == len(rows["ts"]) * len(cols["ts"])


def test_random_store_helper_reproduces_reference_stream():
    z = load_golden("pairs.npz")
    rng = np.random.default_rng(1234)
    r = _ostore(random_store_arrays(rng, 40))
    for k in STORE_FIELDS:
        assert np.array_equal(r[k], z[f"s1234_rows_{k}"])


def test_c9_population_scalar_python_and_c():
    z = load_golden("scalar_c9.npz")
    A, B = c9_population(20_000, 77)
    res = z["res"]
    d = float(z["d"])
    for i in range(0, A.shape[0], 7):  # python scalar on a 1/7 subsample
        got = orc.pair_scalar(tuple(A[i]), tuple(B[i]), d)
        want = None if res[i, 0] != 1.0 else (res[i, 1], res[i, 2])
        assert got == want, i
    for i in range(A.shape[0]):
        got = c_oracle.pair(tuple(A[i]), tuple(B[i]), d)
        want = None if res[i, 0] != 1.0 else (res[i, 1], res[i, 2])
        assert got == want, i


# ── index (index.py:85-188) ───────────────────────────────────────────────


def _index_scenes(z):
    tags = sorted({k.split("_")[0] for k in z.files if k.endswith("_qb")})
    for tag in tags:
        ms = sorted({int(k.split("_")[1][1:]) for k in z.files
                     if k.startswith(tag + "_m") and k.endswith("_hdr")})
        yield tag, ms


def test_index_and_ranges_match_golden():
    z = load_golden("index.npz")
    seen = 0
    for tag, ms in _index_scenes(z):
        st = golden_store(z, tag)
        for m in ms:
            for rule in ("member_extents", "grid_start"):
                key = f"{tag}_m{m}_{rule}"
                ix = orc.index_build(st, m, rule)
                assert [ix["width"], ix["t0"], ix["t_max"]] == list(z[f"{key}_hdr"])
                for f in ("ne_start", "ne_end", "ne_first", "ne_last"):
                    assert np.array_equal(ix[f], z[f"{key}_{f}"]), (key, f)
                assert np.array_equal(ix["nonempty"], z[f"{key}_nonempty"])
                for (b, e), want in zip(zip(z[f"{tag}_qb"], z[f"{tag}_qe"]), z[f"{key}_ranges"]):
                    got = orc.cand_range(ix, float(b), float(e))
                    assert (got is None and want[0] == -1) or tuple(want) == got
                seen += 1
    assert seen >= 20


def test_floor_divide_semantics_numpy_and_c():
    z = load_golden("index.npz")
    a, b, want = z["fd_a"], z["fd_b"], z["fd_res"]
    for ai, bi, wi in zip(a, b, want):
        assert c_oracle.floor_divide(np.array([ai]), float(bi))[0] == wi
    assert np.floor_divide(1.0, 0.1) == 9.0  # not floor(1.0 / 0.1) == 10
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1000, 200_000)
    for w in (0.1, 0.01, 1.0 / 3.0, 0.0999):
        assert np.array_equal(c_oracle.floor_divide(x, w), np.floor_divide(x, w))


# ── planners (planner.py:202-429) ─────────────────────────────────────────


def _table(plan):
    return np.array([(lo, hi, -1 if f is None else f, -1 if l is None else l)
                     for lo, hi, _, _, f, l in plan], dtype=np.int64)


@pytest.mark.parametrize("tag", ["p41", "p47", "p59", "p57"])
def test_planners_match_golden(tag):
    z = load_golden("plans.npz")
    e = golden_store(z, f"{tag}_e")
    q = golden_store(z, f"{tag}_q")
    ix = orc.index_build(e, int(z[f"{tag}_m"]))
    plans = {
        "periodic7": orc.plan_periodic(q, 7, ix),
        "periodic25": orc.plan_periodic(q, 25, ix),
        "fixed1": orc.plan_setsplit_fixed(q, ix, 1),
        "fixed9": orc.plan_setsplit_fixed(q, ix, 9),
        "fixed17": orc.plan_setsplit_fixed(q, ix, 17),
        "minmax3_10": orc.plan_setsplit_minmax(q, ix, 3, 10),
        "minmax5_18": orc.plan_setsplit_minmax(q, ix, 5, 18),
        "max6": orc.plan_setsplit_max(q, ix, 6),
        "max11": orc.plan_setsplit_max(q, ix, 11),
        "gmin4": orc.plan_greedy(q, ix, 4, "min"),
        "gmin8": orc.plan_greedy(q, ix, 8, "min"),
        "gmax4": orc.plan_greedy(q, ix, 4, "max"),
        "gmax8": orc.plan_greedy(q, ix, 8, "max"),
    }
    for name, p in plans.items():
        assert np.array_equal(_table(p), z[f"{tag}_{name}"]), name


# ── engine + brute force (engine.py:151-204, oracle.py:23-41) ─────────────


RES_COLS = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")


def _plan_from_table(tab):
    return [(int(lo), int(hi), None, None, None, None) for lo, hi, _, _ in tab]


@pytest.mark.parametrize("name", ["periodic25", "periodic17", "greedy30", "max40", "single"])
def test_search_small_scene_matches_golden_order_and_stats(name):
    z = load_golden("search.npz")
    e = golden_store(z, "small_e")
    q = golden_store(z, "small_q")
    ix = orc.index_build(e, 60)
    res, st = orc.search(e, ix, q, _plan_from_table(z[f"small_{name}_plan"]), 20.0, workers=3)
    for k in RES_COLS:
        assert np.array_equal(res[k], z[f"small_{name}_{k}"]), k
    assert [st["interactions"], st["temporal_misses"], st["spatial_misses"], st["hits"]] == \
        list(z[f"small_{name}_stats"])
    assert np.array_equal(np.array(st["per_batch"], dtype=np.int64), z[f"small_{name}_per_batch"])


def test_brute_force_small_scene_numpy_and_c():
    z = load_golden("search.npz")
    e = golden_store(z, "small_e")
    q = golden_store(z, "small_q")
    res = orc.brute_force(e, q, 20.0)
    cres, _, _ = c_oracle.brute_force(e, q, 20.0, threads=4)
    for k in RES_COLS:
        assert np.array_equal(res[k], z[f"small_brute_{k}"]), k
        assert np.array_equal(cres[k], z[f"small_brute_{k}"]), k


# ── C engine over spans (the large-scale parity checker) ──────────────────


@pytest.mark.parametrize("name", ["periodic25", "periodic17", "greedy30", "max40", "single"])
def test_c_search_spans_small_scene_matches_golden(name):
    """orc_search_spans (the multi-threaded C engine the scale parity tests
    use) equals the reference's run_search on the golden scenes: items,
    order and per-batch statistics."""
    z = load_golden("search.npz")
    e = golden_store(z, "small_e")
    q = golden_store(z, "small_q")
    tab = z[f"small_{name}_plan"]
    res, pb = c_oracle.search_spans(e, q, tab[:, 0], tab[:, 1], tab[:, 2], tab[:, 3], 20.0, threads=3,
                                    chunk_pairs=997)
    for k in RES_COLS:
        assert np.array_equal(res[k], z[f"small_{name}_{k}"]), k
    stats = z[f"small_{name}_stats"]
    assert [pb[:, 1].sum(), pb[:, 2].sum(), pb[:, 0].sum()] == list(stats[1:])
    per = z[f"small_{name}_per_batch"]
    assert np.array_equal(pb[:, 0], per[:, 4])


@pytest.mark.parametrize("d", [1.0, 5.0])
def test_c_search_spans_config1_matches_golden(d):
    """Config 1 (99,000 × 9,900, m = 10,000, Periodic 120) through the C
    engine on the golden plan table: identical to the reference run."""
    from paper_1405_7461_b200 import datagen

    z = load_golden("search.npz")
    e = datagen.generate_columns(datagen.make_profile("uniform", 1000, seed=1, timesteps=100))
    pool = datagen.generate(datagen.make_profile("uniform", 1000, seed=2, timesteps=100))
    qs = datagen.sample_queries(pool, 100, seed=3)
    E = orc.make_store(*(e[k] for k in STORE_FIELDS))
    Q = orc.make_store(*(getattr(qs, k) for k in STORE_FIELDS))
    tab = z["c1_plan"]
    ix = orc.index_build(E, 10_000)
    f, l = c_oracle.plan_spans(E, ix, Q, tab[:, 0], tab[:, 1])
    assert np.array_equal(f, tab[:, 2]) and np.array_equal(l, tab[:, 3])
    res, pb = c_oracle.search_spans(E, Q, tab[:, 0], tab[:, 1], f, l, d)
    tag = f"c1_d{int(d)}"
    for k in RES_COLS:
        assert np.array_equal(res[k], z[f"{tag}_{k}"]), k
    assert [pb[:, 1].sum(), pb[:, 2].sum(), pb[:, 0].sum()] == list(z[f"{tag}_stats"][1:])


def test_c_search_spans_equals_numpy_oracle_random_scene():
    """Random scene with waypoints and stationary segments, several chunk
    sizes: the C engine equals the numpy restatement item for item."""
    rng = np.random.default_rng(77)
    E = _ostore(random_store_arrays(rng, 3000))
    Q = _ostore(random_store_arrays(rng, 400, first_traj=10_000))
    ix = orc.index_build(E, 50)
    plan = orc.plan_periodic(Q, 23, ix)
    want, st = orc.search(E, ix, Q, plan, 2.5, workers=1)
    lo = np.array([b[0] for b in plan])
    hi = np.array([b[1] for b in plan])
    f, l = c_oracle.plan_spans(E, ix, Q, lo, hi)
    for chunk in (1, 100, 1 << 20):
        got, pb = c_oracle.search_spans(E, Q, lo, hi, f, l, 2.5, threads=4, chunk_pairs=chunk)
        for k in RES_COLS:
            assert np.array_equal(got[k], want[k]), (chunk, k)
        assert pb[:, 1].sum() == st["temporal_misses"] and pb[:, 2].sum() == st["spatial_misses"]


def _extreme_scenes():
    z = load_golden("extreme.npz")
    for tag in z["tags"]:
        yield str(tag), z


def test_extreme_magnitudes_numpy_and_c_match_reference():
    """Overflowing intermediates (|coordinate| 1e150-1e300, d up to 1e300):
    the numpy restatement and the C engine follow the vectorized
    reference, where NaN roots are a miss (core.py:545-553)."""
    import warnings

    for tag, z in _extreme_scenes():
        rows = golden_store(z, f"{tag}_rows")
        cols = golden_store(z, f"{tag}_cols")
        d = float(z[f"{tag}_d"])
        with warnings.catch_warnings(), np.errstate(all="ignore"):
            warnings.simplefilter("ignore")
            ri, ci, tb, te, tm, sm = orc.pair_mesh(rows, cols, d)
        assert np.array_equal(ri, z[f"{tag}_row_idx"]) and np.array_equal(ci, z[f"{tag}_col_idx"]), tag
        assert np.array_equal(tb, z[f"{tag}_t_begin"]) and np.array_equal(te, z[f"{tag}_t_end"]), tag
        assert [tm, sm] == list(z[f"{tag}_misses"]), tag
        nr, nc = rows["ts"].shape[0], cols["ts"].shape[0]
        res, pb = c_oracle.search_spans(rows, cols, [0], [nc - 1], [0], [nr - 1], d, threads=2)
        assert np.array_equal(res["entry_traj"], rows["traj"][z[f"{tag}_row_idx"]]), tag
        assert np.array_equal(res["query_traj"], cols["traj"][z[f"{tag}_col_idx"]]), tag
        assert np.array_equal(res["t_begin"], z[f"{tag}_t_begin"]), tag
        assert np.array_equal(res["t_end"], z[f"{tag}_t_end"]), tag
        assert list(pb[0, 1:]) == list(z[f"{tag}_misses"]), tag
