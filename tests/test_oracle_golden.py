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
