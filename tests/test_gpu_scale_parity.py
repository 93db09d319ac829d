"""Parity at the benchmark's own scale (BASELINE.json configs c2-c5).

The GPU run_search result over a whole plan is compared bit for bit with
the multi-threaded C engine oracle (oracle/pair_oracle.c orc_search_spans,
pinned to the reference's goldens in tests/test_oracle_golden.py):
  c2  Galaxy 1e6 x 40k, in full, at the S1/S2 analogue thresholds
      (hit fractions ~1e-6 and ~2e-4) and
      Periodic s in {60, 120, 240};
  c3  Normal and Normal5 1e7 x 40k, sampled batches, d in {1, 5, 15, 30};
  c4  Exp ~1e7 x ~68k, sampled batches under all six planners;
  c5  Uniform 1e8 x 400k (the headline workload), sampled batches.
Sampling is valid because results are plan-invariant and decompose per
batch (engine.py:176-195): the slice of batch
b in the result is located by the prefix sum of the per-batch hit counts.
"""

from __future__ import annotations

import numpy as np
import pytest

import bench
import paper_1405_7461_b200 as tsk
from helpers import STORE_FIELDS
from oracle import oracle as orc
from oracle.parity import check_batches

pytestmark = pytest.mark.gpu

M = 10_000


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if tsk.device_count() < 1:
        pytest.fail("no CUDA device visible for a -m gpu test")
    tsk.set_device(0)


class Scene:
    def __init__(self, cfg):
        e, q = bench.workload_columns(cfg)
        self.store = tsk.SegmentStore.from_columns(e, validate=False)
        self.queries = tsk.SegmentStore.from_columns(q, validate=False)
        del e, q
        self.index = tsk.build_index(self.store, M)
        self.E = {k: getattr(self.store, k) for k in STORE_FIELDS}  # zero-copy dict views
        self.Q = {k: getattr(self.queries, k) for k in STORE_FIELDS}
        self.oix = orc.index_build(self.E, M)

    def check(self, plan, d, batch_ids=None):
        from paper_1405_7461_b200.engine import search_device

        res, st = tsk.run_search(self.store, self.index, plan, d)
        lo, hi = plan.table()
        hits = np.array([t.hits for t in st.per_batch], np.int64)
        ids = range(len(lo)) if batch_ids is None else batch_ids
        cols = {k: getattr(res, k) for k in orc_res()}
        # per-batch temporal overlaps from the device pipeline (the miss
        # statistics' source) against the oracle's
        ovl = np.asarray(search_device(self.store, self.index, plan, d).per_batch)[:, 2]
        rep = check_batches(self.E, self.oix, self.Q, lo, hi, cols, hits, ids, d, batch_overlaps=ovl)
        assert rep["mismatches"] == 0, rep
        assert rep["overlap_mismatches"] == 0, rep
        # per-batch interactions (engine.py:145) against the oracle's spans
        ints = np.array([t.interactions for t in st.per_batch], np.int64)
        assert rep["pairs"] == int(ints[np.asarray(sorted(set(ids)))].sum())
        return res, st, rep


def orc_res():
    return ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")


def spread(nb, k):
    return sorted(set(np.linspace(0, nb - 1, min(k, nb)).astype(int).tolist()))


_scenes: dict = {}


def scene(name, **over):
    key = (name, tuple(sorted(over.items())))
    if key not in _scenes:
        if len(_scenes) >= 1:  # one large scene resident at a time
            _scenes.clear()
        cfg = dict(bench.CONFIGS[name], **over)
        _scenes[key] = Scene(cfg)
    return _scenes[key]


@pytest.mark.parametrize("s", [60, 120, 240])
@pytest.mark.parametrize("d", [0.15, 1.0])
def test_c2_galaxy_full_plan(d, s):
    """Every batch of c2 (1e6 Galaxy orbits x 40k queries), all stats."""
    sc = scene("c2")
    plan = tsk.periodic(sc.queries, s, sc.index)
    res, st, rep = sc.check(plan, d)
    assert rep["batches"] == len(plan.batches)
    assert st.hits == rep["hits"] == len(res)
    assert (st.temporal_misses, st.spatial_misses) == (rep["temporal_misses"], rep["spatial_misses"])
    assert st.hits > 0
    frac = st.hits / st.interactions_computed
    assert (1e-7 < frac < 1e-5) if d < 0.5 else (5e-5 < frac < 1e-3)


@pytest.mark.parametrize("kind", ["normal", "normal5"])
def test_c3_sampled_threshold_sweep(kind):
    """c3 on Normal and Normal5 start times, d in {1, 5, 15, 30}: 42
    evenly spread batches of the Periodic s = 120 plan per threshold."""
    over = {} if kind == "normal" else {"entries": ("normal5", 25000, 5, 401),
                                        "pool": ("normal5", 1000, 6, 401)}
    sc = scene("c3", **over)
    plan = tsk.periodic(sc.queries, 120, sc.index)
    ids = spread(len(plan.batches), 42)
    for d in (1.0, 5.0, 15.0, 30.0):
        _, st, rep = sc.check(plan, d, ids)
        assert rep["hits"] > 0, d


@pytest.mark.parametrize("planner", sorted(bench.PLANNERS))
def test_c4_sampled_all_planners(planner):
    """c4 (Exp ~1e7 x ~68k, d = 5) under each of the six planners of the
    paper's comparison (Table 3): 16 evenly spread batches."""
    sc = scene("c4")
    plan = bench.PLANNERS[planner](tsk, sc.queries, sc.index)
    _, st, rep = sc.check(plan, 5.0, spread(len(plan.batches), 16))
    assert rep["hits"] > 0


def test_c5_headline_sampled():
    """c5, the headline (Uniform 1e8 x 400k, d = 1, Periodic 120): 12 evenly
    spread batches (~1.1e9 pairs) through the oracle, bit for bit."""
    sc = scene("c5")
    plan = tsk.periodic(sc.queries, 120, sc.index)
    _, st, rep = sc.check(plan, 1.0, spread(len(plan.batches), 12))
    assert rep["hits"] > 0 and rep["pairs"] > 5e8
