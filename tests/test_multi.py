"""Multi-GPU sharding: host logic on CPU with gloo, world 2.

The batch plan is cut into contiguous interaction-balanced shards, each rank
evaluates its shard against its replica of the store (here the CPU oracle
stands in for the GPU), and the shard-ordered concatenation must equal the
single-device result bit for bit, order and statistics included.  A GPU test
runs the library's own sharded path (``run_search(..., devices=[0, 0])``).
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1405_7461_b200 as tsk
from paper_1405_7461_b200.sharding import batch_interactions, shard_bounds, sub_plan

RES = ("query_traj", "query_seg", "entry_traj", "entry_seg", "t_begin", "t_end")
FIELDS = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")


def _scene():
    from test_host import host_index

    store = tsk.generate(tsk.make_profile("uniform", 60, seed=41, timesteps=80))
    pool = tsk.generate(tsk.make_profile("uniform", 30, seed=42, timesteps=80))
    q = tsk.sample_queries(pool, 5, seed=43)
    ix = host_index(store, 200)
    return store, ix, q, tsk.periodic(q, 23, ix)


def _oracle_run(store, ix_store, plan, d):
    from oracle import oracle as orc

    e = {k: getattr(store, k) for k in FIELDS}
    q = {k: getattr(plan.queries, k) for k in FIELDS}
    oix = orc.index_build(e, 200)
    oplan = [(b.lo, b.hi, None, None, None, None) for b in plan.batches]
    return orc.search(e, oix, q, oplan, d, workers=2)


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    store, ix, q, plan = _scene()
    bounds = shard_bounds(batch_interactions(plan, ix), world)
    b0, b1 = bounds[rank]
    sp = sub_plan(plan, b0, b1)
    res, st = _oracle_run(store, ix, sp, 9.0) if sp is not None else (None, None)
    gathered = [None] * world
    dist.all_gather_object(gathered, (b0, b1, res, st))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_bounds_are_contiguous_and_balanced():
    ints = np.array([5, 0, 9, 3, 3, 3, 20, 1, 1, 1], dtype=np.int64)
    for world in (1, 2, 3, 4, 8, 16):
        b = shard_bounds(ints, world)
        assert b[0][0] == 0 and b[-1][1] == len(ints)
        assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
        assert all(x0 <= x1 for x0, x1 in b)
    b = shard_bounds(np.full(100, 7, dtype=np.int64), 4)
    assert [x1 - x0 for x0, x1 in b] == [25, 25, 25, 25]


def test_gloo_world2_sharded_equals_single():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = out.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    store, ix, q, plan = _scene()
    want, wst = _oracle_run(store, ix, plan, 9.0)
    parts = [g for g in gathered if g[2] is not None]
    assert [g[0] for g in gathered] == sorted(g[0] for g in gathered)
    for k in RES:
        got = np.concatenate([g[2][k] for g in parts])
        assert np.array_equal(got, want[k]), k
    for key in ("interactions", "temporal_misses", "spatial_misses", "hits"):
        assert sum(g[3][key] for g in parts) == wst[key]
    # per-batch interactions (rebased ordinals) line up with the whole plan
    pb = [row[3] for g in parts for row in g[3]["per_batch"]]
    assert pb == [row[3] for row in wst["per_batch"]]


@pytest.mark.gpu
def test_library_sharded_run_search_equals_single_device():
    if tsk.device_count() < 1:
        pytest.fail("no CUDA device")
    store = tsk.generate(tsk.make_profile("uniform", 300, seed=51, timesteps=120))
    pool = tsk.generate(tsk.make_profile("uniform", 60, seed=52, timesteps=120))
    q = tsk.sample_queries(pool, 12, seed=53)
    ix = tsk.build_index(store, 2000)
    plan = tsk.periodic(q, 60, ix)
    base, bst = tsk.run_search(store, ix, plan, 6.0)
    for devs in ([0, 0], [0, 0, 0]):
        res, st = tsk.run_search(store, ix, plan, 6.0, devices=devs)
        for k in RES:
            assert np.array_equal(getattr(res, k), getattr(base, k)), k
        assert (st.interactions_computed, st.temporal_misses, st.spatial_misses, st.hits) == \
            (bst.interactions_computed, bst.temporal_misses, bst.spatial_misses, bst.hits)
        assert [t.interactions for t in st.per_batch] == [t.interactions for t in bst.per_batch]


def _gpu_worker(rank, world, port, out):
    """One rank of the bench's N>1 layout on the GPU library: each rank
    uploads its own replica of the store (as under torchrun; in one process
    replicas are device-to-device copies, tsk_db_replicate), the plan is cut
    into interaction-balanced shards, each rank runs run_search on its shard,
    and gloo carries the results back."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tsk.set_device(0)  # both ranks on the one GPU of the box
    store, _, q, _ = _scene()
    ix = tsk.build_index(store, 200)
    plan = tsk.periodic(q, 23, ix)
    bounds = shard_bounds(batch_interactions(plan, ix), world)
    b0, b1 = bounds[rank]
    sp = sub_plan(plan, b0, b1)
    part = None
    if sp is not None:
        res, st = tsk.run_search(store, ix, sp, 9.0)
        part = ({k: np.asarray(getattr(res, k)).copy() for k in RES},
                (st.interactions_computed, st.temporal_misses, st.spatial_misses, st.hits))
    gathered = [None] * world
    dist.all_gather_object(gathered, (b0, b1, part))
    if rank == 0:
        out.put(gathered)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_gpu_ranks_equal_oracle():
    """The sharded N>1 path with the GPU library in every rank (both ranks on
    GPU 0 of a one-GPU box): the shard-ordered concatenation equals the CPU
    oracle's single run bit for bit, statistics included."""
    if tsk.device_count() < 1:
        pytest.fail("no CUDA device")
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    gathered = out.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    store, ix, q, plan = _scene()
    want, wst = _oracle_run(store, ix, plan, 9.0)
    parts = [g[2] for g in sorted(gathered, key=lambda g: g[0]) if g[2] is not None]
    assert len(parts) == 2
    for k in RES:
        assert np.array_equal(np.concatenate([p[0][k] for p in parts]), want[k]), k
    tot = np.sum([p[1] for p in parts], axis=0)
    assert tuple(int(x) for x in tot) == (wst["interactions"], wst["temporal_misses"], wst["spatial_misses"],
                                           wst["hits"])
