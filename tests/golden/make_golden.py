"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference `trajseek` from /root/reference/pkg/src and
writes small .npz fixtures next to this file.  The fixtures are
committed; nothing on the GPU box reads /root/reference.

What is pinned (reference file:line in each section):
  pairs_*.npz     core.pair_intervals (core.py:464-565) incl. hand cases
                  from tests/test_core.py:49-155 and the 40x55 seed-1234
                  scene of tests/test_core.py:249-265
  scalar_c9.npz   core.threshold_interval on C9-style pairs
                  (tests/test_acceptance.py:319-407), 20k pairs
  index_*.npz     index.build_index / candidate_range (index.py:85-173)
  plans.npz       all six planners on random scenes (planner.py:202-429)
  search_*.npz    engine.run_search results + stats (engine.py:151-204)
  brute_*.npz     oracle.brute_force_search (oracle.py:23-41)
  datagen.npz     sha256 of datagen.generate/sample_queries outputs
"""

from __future__ import annotations

import hashlib
import math
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))  # tests/ for helpers

import trajseek  # noqa: E402  (the reference)
from trajseek import core, datagen, engine, index, oracle, planner  # noqa: E402

from helpers import STORE_FIELDS, c9_population, random_store_arrays, store_digest  # noqa: E402


def ref_store(arr):
    return core.SegmentStore(*(arr[k] for k in STORE_FIELDS))


def store_arrays(s):
    return {k: np.asarray(getattr(s, k)).copy() for k in STORE_FIELDS}


def save(name, **kw):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **kw)
    print("wrote", path, os.path.getsize(path), "bytes")


def flat_store(prefix, arr, out):
    for k in STORE_FIELDS:
        out[f"{prefix}_{k}"] = arr[k]


# ── pairs ───────────────────────────────────────────────────────────────────


def hand_cases():
    """The hand-derived pairs of tests/test_core.py:49-155 as 8-tuples."""
    S = lambda *v: tuple(float(x) for x in v)  # xs ys zs ts xe ye ze te
    return [
        (S(0, 0, 0, 0, 0, 0, 0, 1), S(10, 0, 0, 0, -10, 0, 0, 1), 1.0),
        (S(0, 0, 0, 2, 0, 0, 0, 5), S(3, 0, 0, 2, 3, 0, 0, 5), 5.0),
        (S(0, 0, 0, 2, 0, 0, 0, 5), S(3, 0, 0, 2, 3, 0, 0, 5), 3.0),
        (S(0, 0, 0, 2, 0, 0, 0, 5), S(3, 0, 0, 2, 3, 0, 0, 5), 2.999),
        (S(0, 0, 0, 0, 4, 0, 0, 4), S(0, 2, 0, 0, 4, 2, 0, 4), 2.0),
        (S(0, 0, 0, 0, 4, 0, 0, 4), S(0, 2, 0, 0, 4, 2, 0, 4), 1.0),
        (S(0, 0, 0, 0, 0, 0, 0, 2), S(-1, 3, 0, 0, 1, 3, 0, 2), 3.0),
        (S(0, 0, 0, 0, 0, 0, 0, 2), S(-1, 3, 0, 0, 1, 3, 0, 2), 2.9),
        (S(0, 0, 0, 3, 0, 0, 0, 3), S(0, 4, 0, 3, 0, 4, 0, 3), 4.0),
        (S(0, 0, 0, 3, 0, 0, 0, 3), S(0, 4, 0, 3, 0, 4, 0, 3), 3.9),
        (S(0, 0, 0, 0, 0, 0, 0, 1), S(0.5, 0, 0, 0, 20, 0, 0, 1), 1.0),
        (S(0, 0, 0, 0, 2, 0, 0, 2), S(2, 0, 0, 0, 0, 0, 0, 2), 0.0),
        (S(0, 0, 0, 0, 10, 0, 0, 10), S(0, 1, 0, 4, 0, 1, 0, 6), 1.5),
        (S(0.1, 0.2, 0.3, 1, 0.7, 0.8, 0.9, 3), S(0, 0, 0, 1, 0, 0, 0, 3), 1.0),
        (S(0, 0, 0, 0, 0, 0, 0, 1), S(0, 0, 0, 1.5, 0, 0, 0, 2), 100.0),
        (S(0, 0, 0, 0, 6, 0, 0, 2), S(6, 0, 0, 2, 9, 0, 0, 4), 0.5),
        # touching extents where the clip lands on an end point that the
        # lerp would not reproduce exactly (S + (E - S) != E)
        (S(1.0, 0, 0, 0, 1e-17, 0, 0, 1), S(0, 0, 0, 1, 5, 0, 0, 2), 1.0),
        (S(0, 0, 0, 1, 5, 0, 0, 2), S(1.0, 0, 0, 0, 1e-17, 0, 0, 1), 1.0),
        # waypoint at the end of the other segment
        (S(3, 4, 0, 5, 9, 9, 9, 5), S(0, 0, 0, 1, 3, 4, 0, 5), 0.0),
    ]


def gen_pairs():
    out = {}
    cases = hand_cases()
    rows = np.array([c[0] for c in cases])
    cols = np.array([c[1] for c in cases])
    ds = np.array([c[2] for c in cases])
    res = []
    for a, b, d in cases:
        iv = core.threshold_interval(*core.temporal_intersection(_seg(a), _seg(b)), d) \
            if core.temporal_intersection(_seg(a), _seg(b)) is not None else None
        res.append((1.0, iv.begin, iv.end) if iv is not None else (0.0, 0.0, 0.0))
    out["hand_a"] = rows
    out["hand_b"] = cols
    out["hand_d"] = ds
    out["hand_res"] = np.array(res)

    # 40x55 scene, seed 1234, d=4 (tests/test_core.py:249-265) and more
    for tag, seed, nr, nc, d in (("s1234", 1234, 40, 55, 4.0), ("s99", 99, 30, 30, 2.0),
                                 ("s7", 7, 200, 150, 3.0), ("s8", 8, 120, 333, 0.0)):
        rng = np.random.default_rng(seed)
        r = random_store_arrays(rng, nr)
        c = random_store_arrays(rng, nc, first_traj=1000)
        hits = core.pair_intervals(ref_store(r), ref_store(c), d)
        flat_store(f"{tag}_rows", store_arrays(ref_store(r)), out)
        flat_store(f"{tag}_cols", store_arrays(ref_store(c)), out)
        out[f"{tag}_d"] = np.float64(d)
        out[f"{tag}_row_idx"] = hits.row_idx
        out[f"{tag}_col_idx"] = hits.col_idx
        out[f"{tag}_t_begin"] = hits.t_begin
        out[f"{tag}_t_end"] = hits.t_end
        out[f"{tag}_misses"] = np.array([hits.temporal_misses, hits.spatial_misses])
    save("pairs.npz", **out)


def _seg(v):
    return core.TrajectorySegment(0, 0, core.SpacetimePoint(*v[0:4]), core.SpacetimePoint(*v[4:8]))


def gen_scalar_c9():
    """C9-style pair population (tests/test_acceptance.py:319-345), 20k pairs.
    Inputs are regenerated from the seed by helpers.c9_population."""
    A, B = c9_population(20_000, 77)
    n = A.shape[0]
    res = np.zeros((n, 3))
    for i in range(n):
        clip = core.temporal_intersection(_seg(A[i]), _seg(B[i]))
        if clip is None:
            res[i] = (-1.0, 0.0, 0.0)
            continue
        iv = core.threshold_interval(clip[0], clip[1], 1.0)
        if iv is not None:
            res[i] = (1.0, iv.begin, iv.end)
    save("scalar_c9.npz", d=np.float64(1.0), res=res)


# ── index / ranges ──────────────────────────────────────────────────────────


def gen_index():
    out = {}
    scenes = []
    rng = np.random.default_rng(21)
    scenes.append(("r300", random_store_arrays(rng, 300), (1, 7, 33, 128)))
    rng = np.random.default_rng(22)
    scenes.append(("r400", random_store_arrays(rng, 400), (1, 5, 40, 500)))
    up = datagen.generate(datagen.make_profile("uniform", 40, seed=4, timesteps=60))
    scenes.append(("u40", store_arrays(up), (10, 1000, 10_000)))
    ex = datagen.generate(datagen.make_profile("exp", 40, seed=9))
    scenes.append(("e40", store_arrays(ex), (64, 10_000)))
    for tag, arr, ms in scenes:
        st = ref_store(arr)
        flat_store(tag, store_arrays(st), out)
        qrng = np.random.default_rng(5)
        lo_t, hi_t = float(st.ts.min()) - 1.0, float(st.te.max()) + 1.0
        b = qrng.uniform(lo_t, hi_t, 300)
        e = b + qrng.uniform(0.0, (hi_t - lo_t) / 10.0, 300)
        out[f"{tag}_qb"] = b
        out[f"{tag}_qe"] = e
        for m in ms:
            for rule in ("member_extents", "grid_start"):
                ix = index.build_index(st, m, extent_rule=rule)
                key = f"{tag}_m{m}_{rule}"
                out[f"{key}_hdr"] = np.array([ix.bin_width, ix.t0, ix.t_max])
                out[f"{key}_ne_start"] = ix._ne_start
                out[f"{key}_ne_end"] = ix._ne_end
                out[f"{key}_ne_first"] = ix._ne_first
                out[f"{key}_ne_last"] = ix._ne_last
                out[f"{key}_nonempty"] = np.array([not bb.empty for bb in ix.bins])
                rr = []
                for bi, ei in zip(b, e):
                    sp = index.candidate_range(ix, core.TimeInterval(float(bi), float(ei)))
                    rr.append((-1, -1) if sp is None else sp)
                out[f"{key}_ranges"] = np.array(rr, dtype=np.int64)
    # floor_divide corner cases used by bin assignment
    a = np.array([1.0, 0.3, 0.7, 2.9999999999999996, 3.0, 1e-300, 5.551115123125783e-17, 99.99999999999999])
    out["fd_a"] = a
    out["fd_b"] = np.array([0.1, 0.1, 0.1, 0.3, 0.3, 0.1, 0.1, 0.01])
    out["fd_res"] = np.floor_divide(a, out["fd_b"])
    save("index.npz", **out)


# ── planners ────────────────────────────────────────────────────────────────


def plan_table(plan):
    return np.array([(b.lo, b.hi, -1 if b.first is None else b.first,
                      -1 if b.last is None else b.last) for b in plan.batches], dtype=np.int64)


def gen_plans():
    out = {}
    for tag, seed, ne, nq, m in (("p41", 41, 300, 80, 16), ("p47", 47, 300, 96, 16),
                                 ("p59", 59, 220, 66, 14), ("p57", 57, 350, 90, 6)):
        rng = np.random.default_rng(seed)
        e = random_store_arrays(rng, ne)
        q = random_store_arrays(rng, nq, first_traj=10_000)
        es, qs = ref_store(e), ref_store(q)
        ix = index.build_index(es, m)
        flat_store(f"{tag}_e", store_arrays(es), out)
        flat_store(f"{tag}_q", store_arrays(qs), out)
        out[f"{tag}_m"] = np.int64(m)
        plans = {
            "periodic7": planner.periodic(qs, 7, ix),
            "periodic25": planner.periodic(qs, 25, ix),
            "fixed1": planner.setsplit_fixed(qs, ix, 1),
            "fixed9": planner.setsplit_fixed(qs, ix, 9),
            "fixed17": planner.setsplit_fixed(qs, ix, 17),
            "minmax3_10": planner.setsplit_minmax(qs, ix, 3, 10),
            "minmax5_18": planner.setsplit_minmax(qs, ix, 5, 18),
            "max6": planner.setsplit_max(qs, ix, 6),
            "max11": planner.setsplit_max(qs, ix, 11),
            "gmin4": planner.greedy_min(qs, ix, 4),
            "gmin8": planner.greedy_min(qs, ix, 8),
            "gmax4": planner.greedy_max(qs, ix, 4),
            "gmax8": planner.greedy_max(qs, ix, 8),
        }
        for name, p in plans.items():
            out[f"{tag}_{name}"] = plan_table(p)
    save("plans.npz", **out)


# ── engine / brute force ───────────────────────────────────────────────────


def result_arrays(res, prefix, out):
    for k in ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end"):
        out[f"{prefix}_{k}"] = np.asarray(getattr(res, k))


def stats_arrays(st, prefix, out):
    out[f"{prefix}_stats"] = np.array([st.interactions_computed, st.temporal_misses,
                                       st.spatial_misses, st.hits], dtype=np.int64)
    out[f"{prefix}_per_batch"] = np.array(
        [(t.ordinal, t.queries, t.candidates, t.interactions, t.hits) for t in st.per_batch],
        dtype=np.int64)


def gen_search():
    out = {}
    # small_scene of the reference conftest (tests/conftest.py:38-49)
    store = datagen.generate(datagen.make_profile("uniform", 6, seed=3, timesteps=150))
    pool = datagen.generate(datagen.make_profile("uniform", 6, seed=8, timesteps=150))
    qs = datagen.sample_queries(pool, 2, seed=11)
    flat_store("small_e", store_arrays(store), out)
    flat_store("small_q", store_arrays(qs), out)
    ix = index.build_index(store, 60)
    for name, plan in (("periodic25", planner.periodic(qs, 25, ix)),
                       ("periodic17", planner.periodic(qs, 17, ix)),
                       ("greedy30", planner.greedy_min(qs, ix, 30)),
                       ("max40", planner.setsplit_max(qs, ix, 40)),
                       ("single", planner.periodic(qs, len(qs), ix))):
        res, st = engine.run_search(store, ix, plan, 20.0, workers=1)
        result_arrays(res, f"small_{name}", out)
        stats_arrays(st, f"small_{name}", out)
        out[f"small_{name}_plan"] = plan_table(plan)
    bf = oracle.brute_force_search(store, qs, 20.0)
    result_arrays(bf, "small_brute", out)

    # config 1: uniform 1000x100, queries 100 of pool seed 2, m=10k, s=120
    store = datagen.generate(datagen.make_profile("uniform", 1000, seed=1, timesteps=100))
    pool = datagen.generate(datagen.make_profile("uniform", 1000, seed=2, timesteps=100))
    qs = datagen.sample_queries(pool, 100, seed=3)
    out["c1_e_digest"] = np.frombuffer(store_digest(store_arrays(store)), np.uint8)
    out["c1_q_digest"] = np.frombuffer(store_digest(store_arrays(qs)), np.uint8)
    ix = index.build_index(store, 10_000)
    plan = planner.periodic(qs, 120, ix)
    out["c1_plan"] = plan_table(plan)
    for d in (1.0, 5.0):
        res, st = engine.run_search(store, ix, plan, d, workers=1)
        result_arrays(res, f"c1_d{int(d)}", out)
        stats_arrays(st, f"c1_d{int(d)}", out)
    save("search.npz", **out)


def gen_datagen():
    out = {}
    cases = [("uniform", 5, 3, {}), ("normal", 7, 4, {}), ("normal5", 9, 5, {}),
             ("exp", 30, 6, {}), ("uniform", 3, 7, {"timesteps": 20, "step_scale": 2.5})]
    for i, (kind, n, seed, kw) in enumerate(cases):
        s = datagen.generate(datagen.make_profile(kind, n, seed=seed, **kw))
        out[f"g{i}"] = np.frombuffer(store_digest(store_arrays(s)), np.uint8)
        out[f"g{i}_n"] = np.int64(len(s))
        q = datagen.sample_queries(s, max(1, n // 2), seed=seed + 100)
        out[f"g{i}_q"] = np.frombuffer(store_digest(store_arrays(q)), np.uint8)
    save("datagen.npz", **out)


def gen_csv():
    """datagen.save / load (datagen.py:273-333) and the CLI result CSV
    (cli.py:62-77), written by the reference itself."""
    import json
    import tempfile

    from trajseek.cli import main as cli_main

    store = datagen.generate(datagen.make_profile("uniform", 5, seed=3, timesteps=40))
    datagen.save(store, os.path.join(HERE, "store_uniform.csv"))
    ex = datagen.generate(datagen.make_profile("exp", 12, seed=6))
    datagen.save(ex, os.path.join(HERE, "store_exp.csv"))
    with tempfile.TemporaryDirectory() as td:
        db, pool, qf = (os.path.join(td, n) for n in ("db.csv", "pool.csv", "q.csv"))
        assert cli_main(["gen", "--profile", "uniform", "--trajectories", "12", "--seed", "5",
                         "--out", db]) == 0
        assert cli_main(["gen", "--profile", "uniform", "--trajectories", "8", "--seed", "6",
                         "--out", pool]) == 0
        assert cli_main(["gen", "--sample-from", pool, "--trajectories", "2", "--seed", "7",
                         "--out", qf]) == 0
        for sorted_flag, name in ((True, "results_sorted.csv"), (False, "results_engine.csv")):
            args = ["search", "--db", db, "--queries", qf, "--d", "20.0", "--m", "60",
                    "--workers", "1", "--planner", "greedy-max", "--bound", "50",
                    "--out", os.path.join(HERE, name)]
            if sorted_flag:
                args.insert(-2, "--sorted")
            assert cli_main(args) == 0
        json.dump({"cli_db.csv": hashlib.sha256(open(db, "rb").read()).hexdigest(),
                   "cli_queries.csv": hashlib.sha256(open(qf, "rb").read()).hexdigest()},
                  open(os.path.join(HERE, "cli_inputs_sha256.json"), "w"), indent=1)
        # load() error messages for malformed files
        errs = {}
        good = open(os.path.join(HERE, "store_uniform.csv")).read().splitlines()
        cases = {
            "bad_header": ["a,b,c"] + good[1:3],
            "arity": good[:2] + ["1,2,3"],
            "nonnumeric": good[:2] + ["1,0,abc,0,0,0,1,0,0,1"],
            "nonfinite": good[:2] + ["1,0,inf,0,0,0,1,0,0,1"],
            "reversed": good[:2] + ["1,0,0,0,0,5.0,1,0,0,1.5"],
            "unsorted_strict": good[:1] + [good[3], good[2]],
            "empty_rows": good[:1],
        }
        for name, lines in cases.items():
            path = os.path.join(td, name + ".csv")
            open(path, "w").write("\n".join(lines) + "\n")
            try:
                datagen.load(path, strict=(name == "unsorted_strict"))
                errs[name] = {"lines": lines, "error": None}
            except core.FormatError as exc:
                errs[name] = {"lines": lines, "error": str(exc).replace(path, "<path>")}
        json.dump(errs, open(os.path.join(HERE, "load_errors.json"), "w"), indent=1)
    print("wrote csv fixtures")


if __name__ == "__main__":
    print("reference trajseek", trajseek.__version__, "from", trajseek.__file__)
    gen_pairs()
    gen_scalar_c9()
    gen_index()
    gen_plans()
    gen_search()
    gen_datagen()
    gen_csv()
