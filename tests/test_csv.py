"""CSV I/O parity with the reference (datagen.py:273-333, cli.py:62-77).

Golden files were written by the reference itself (tests/golden/make_golden.py):
datagen.save output, the CLI's search result CSV (sorted and engine order),
load() error messages, and digests of the CLI's generated inputs.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1405_7461_b200 as tsk
from helpers import GOLDEN, STORE_FIELDS
from paper_1405_7461_b200 import _native


def test_native_repr_matches_python_repr():
    rng = np.random.default_rng(0)
    bits = rng.integers(0, 2**63, 200_000, dtype=np.int64).astype(np.uint64)
    bits |= rng.integers(0, 2, 200_000).astype(np.uint64) << np.uint64(63)
    xs = bits.view(np.float64)
    xs = np.concatenate([xs[np.isfinite(xs)], rng.uniform(-1e3, 1e3, 50_000),
                         np.round(rng.uniform(-1e6, 1e6, 50_000), 3),
                         [0.0, -0.0, 1e16, 1e-5, 1e-4, 9999999999999998.0, 5e-324, 1.7976931348623157e308,
                          -1.7976931348623157e308, 0.1, 0.30000000000000004, 123.0, 1e22]])
    bad = [x for x in xs if _native.py_repr(float(x)) != repr(float(x))]
    assert bad == []


@pytest.mark.parametrize("name,kind,n,seed,kw", [
    ("store_uniform.csv", "uniform", 5, 3, {"timesteps": 40}),
    ("store_exp.csv", "exp", 12, 6, {}),
])
def test_save_is_byte_identical_to_reference(tmp_path, name, kind, n, seed, kw):
    store = tsk.generate(tsk.make_profile(kind, n, seed=seed, **kw))
    out = tmp_path / name
    tsk.save(store, str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


def test_load_round_trip_and_reference_file(tmp_path):
    s = tsk.load(os.path.join(GOLDEN, "store_exp.csv"))
    ref = tsk.generate(tsk.make_profile("exp", 12, seed=6))
    for k in STORE_FIELDS:
        assert np.array_equal(getattr(s, k), getattr(ref, k))
    out = tmp_path / "again.csv"
    tsk.save(s, str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, "store_exp.csv"), "rb").read()


def test_cli_inputs_reproduce_reference_digests(tmp_path):
    want = json.load(open(os.path.join(GOLDEN, "cli_inputs_sha256.json")))
    db = tsk.generate(tsk.make_profile("uniform", 12, seed=5))
    pool = tsk.generate(tsk.make_profile("uniform", 8, seed=6))
    q = tsk.sample_queries(pool, 2, seed=7)
    for store, name in ((db, "cli_db.csv"), (q, "cli_queries.csv")):
        p = tmp_path / name
        tsk.save(store, str(p))
        assert hashlib.sha256(p.read_bytes()).hexdigest() == want[name], name


def test_load_errors_match_reference_messages(tmp_path):
    cases = json.load(open(os.path.join(GOLDEN, "load_errors.json")))
    for name, case in cases.items():
        path = tmp_path / f"{name}.csv"
        path.write_text("\n".join(case["lines"]) + "\n")
        if case["error"] is None:
            tsk.load(str(path), strict=(name == "unsorted_strict"))
            continue
        with pytest.raises(tsk.FormatError) as exc:
            tsk.load(str(path), strict=(name == "unsorted_strict"))
        assert str(exc.value).replace(str(path), "<path>") == case["error"], name


def test_load_unsorted_rows_are_sorted_stably(tmp_path):
    lines = open(os.path.join(GOLDEN, "store_uniform.csv")).read().splitlines()
    body = lines[1:]
    rng = np.random.default_rng(3)
    perm = rng.permutation(len(body))
    p = tmp_path / "shuffled.csv"
    p.write_text("\n".join([lines[0]] + [body[i] for i in perm]) + "\n")
    s = tsk.load(str(p))
    ref = tsk.generate(tsk.make_profile("uniform", 5, seed=3, timesteps=40))
    assert np.array_equal(np.sort(s.ts), ref.ts)
    assert np.all(np.diff(s.ts) >= 0)
    with pytest.raises(tsk.FormatError):
        tsk.load(str(p), strict=True)


def test_result_csv_writer_formats_like_the_cli(tmp_path):
    # the reference CLI's sorted result file, re-emitted from its parsed rows
    src = open(os.path.join(GOLDEN, "results_sorted.csv")).read()
    rows = [r.split(",") for r in src.splitlines()[1:]]
    res = tsk.ResultSet(*[np.array([int(r[k]) for r in rows]) for k in range(4)],
                        *[np.array([float(r[k]) for r in rows]) for k in (4, 5)])
    out = tmp_path / "res.csv"
    tsk.write_results(res, str(out))
    assert out.read_text() == src
    tsk.write_results(tsk.ResultSet.empty(), str(out))
    assert out.read_text() == "query_traj,query_seg,entry_traj,entry_seg,t_begin,t_end\n"


@pytest.mark.gpu
def test_search_result_csv_is_byte_identical_to_reference_cli(tmp_path):
    """cli `search --sorted` and engine-order output (cli.py:217-227) reproduced
    end to end: same inputs, GPU search, native writer."""
    db = tsk.generate(tsk.make_profile("uniform", 12, seed=5))
    pool = tsk.generate(tsk.make_profile("uniform", 8, seed=6))
    q = tsk.sample_queries(pool, 2, seed=7)
    # the CLI reloads its CSV inputs: round-trip them the same way
    tsk.save(db, str(tmp_path / "db.csv"))
    tsk.save(q, str(tmp_path / "q.csv"))
    db = tsk.load(str(tmp_path / "db.csv"))
    q = tsk.load(str(tmp_path / "q.csv"))
    ix = tsk.build_index(db, 60)
    plan = tsk.greedy_max(q, ix, 50)
    res, _ = tsk.run_search(db, ix, plan, 20.0)
    for canonical, name in ((True, "results_sorted.csv"), (False, "results_engine.csv")):
        out = tmp_path / name
        tsk.write_results(res, str(out), canonical=canonical)
        assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read(), name
