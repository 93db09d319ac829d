"""Benchmark: distance-threshold search throughput (segment-pair evals/s) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 ... bench.py --gpus N

A step is one pass of the hot path over the workload's batch plan:
  * value — device throughput with the queries resident in HBM and hits left
    in HBM: Σ interactions ÷ CUDA-event time of the search pipeline
    (K3 ranges → K1 pair kernel → K4 sort/gather), max over ranks.
  * e2e — the same metric through the public drop-in call
    ``run_search(store, index, plan, d)`` with pinned host query columns:
    H2D of the queries and D2H of the ResultSet inside the timed region
    (the reference's "response time"; DB resident).
The entry store is replicated on every GPU and the batch plan is sharded
into contiguous, interaction-balanced slices (no collective on the data
path; NCCL only carries the timing max).

--impl reference times the reference's CPU algorithm (the numpy port in
oracle/ — the reference is pure Python + numpy and cannot travel to the
GPU box) on sampled batches of the same workload on all host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "distance-threshold query response time; segment-pair evals/s @1/2/4/8 B200"
UNIT = "pair-evals/s"

# Workloads of BASELINE.json "configs".  Entries / query pool:
# (profile kind, trajectories, seed, timesteps) through the reference datagen stream.
CONFIGS = {
    "c1": dict(desc="RandWalk-Uniform 1,000x100 (99,000 entries), 100 query trajectories "
                    "(9,900 query segments), d=5, Periodic s=120, m=10,000",
               entries=("uniform", 1000, 1, 100), pool=("uniform", 1000, 2, 100), sample=(100, 3),
               d=5.0),
    "c2": dict(desc="Galaxy-shaped star orbits 2,500x401 (1,000,000 entries), 100 orbit "
                    "trajectories (40,000 query segments), d=0.5, Periodic s=120, m=10,000",
               galaxy=(2500, 11), galaxy_pool=(400, 12), sample=(100, 13), d=0.5),
    "c3": dict(desc="RandWalk-Normal 25,000x401 (1e7 entries), 100 query trajectories "
                    "(40,000 query segments), d=5, Periodic s=120, m=10,000",
               entries=("normal", 25000, 5, 401), pool=("normal", 1000, 6, 401), sample=(100, 7),
               d=5.0),
    "c4": dict(desc="RandWalk-Exp 140,000 trajectories (~1e7 entries), 1,000 query trajectories, "
                    "d=5, Periodic s=120, m=10,000",
               entries=("exp", 140000, 8, None), pool=("exp", 14000, 9, None), sample=(1000, 10),
               d=5.0),
    "c5": dict(desc="RandWalk-Uniform 250,000x401 (1e8 entries), 1,000 query trajectories "
                    "(400,000 query segments), d=1, Periodic s=120, m=10,000",
               entries=("uniform", 250000, 21, 401), pool=("uniform", 1000, 22, 401), sample=None,
               d=1.0),
}
S_BATCH = 120
M_BINS = 10_000

# Planner settings of config 4: s = 120 throughout.
PLANNERS = {
    "periodic": lambda tsk, q, ix: tsk.periodic(q, S_BATCH, ix),
    "setsplit_fixed": lambda tsk, q, ix: tsk.setsplit_fixed(q, ix, -(-len(q) // S_BATCH)),
    "setsplit_max": lambda tsk, q, ix: tsk.setsplit_max(q, ix, S_BATCH),
    "setsplit_minmax": lambda tsk, q, ix: tsk.setsplit_minmax(q, ix, 16, S_BATCH),
    "greedy_min": lambda tsk, q, ix: tsk.greedy_min(q, ix, S_BATCH),
    "greedy_max": lambda tsk, q, ix: tsk.greedy_max(q, ix, S_BATCH),
}
W_DECIDE, W_HIT = 50, 9  # FP64 flops per overlapping pair / extra per hit
F32_OPS = 10.25  # FP32 pre-filter ops per evaluated pair: 6 separation + 3 norm, plus per (query, lane) of 4 pairs 2 threshold + 2 min + 1 compare


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ── workload construction ───────────────────────────────────────────────────


def workload_columns(cfg):
    """(entries, queries) as unsorted column dicts — identical on every rank/arm."""
    from paper_1405_7461_b200 import datagen

    if "galaxy" in cfg:
        e = datagen.galaxy(*cfg["galaxy"])
        pool = datagen.galaxy(*cfg["galaxy_pool"])
        q = datagen.sample_queries(pool, *cfg["sample"])
        cols = lambda s: {k: getattr(s, k) for k in ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")}  # noqa: E731
        return cols(e), cols(q)

    def prof(spec):
        kind, n, seed, steps = spec
        kw = {} if steps is None else {"timesteps": steps}
        return datagen.make_profile(kind, n, seed=seed, **kw)

    e = datagen.generate_columns(prof(cfg["entries"]))
    p = datagen.generate_columns(prof(cfg["pool"]))
    if cfg["sample"] is not None:
        n, seed = cfg["sample"]
        ids = np.unique(p["traj"])
        pick = np.random.default_rng(seed).choice(ids, size=n, replace=False)
        keep = np.isin(p["traj"], pick)
        p = {k: v[keep] for k, v in p.items()}
    return e, p


FIELDS = ("traj", "seg", "xs", "ys", "zs", "ts", "xe", "ye", "ze", "te")


from paper_1405_7461_b200.sharding import shard_bounds, sub_plan  # noqa: E402


# ── clocks ──────────────────────────────────────────────────────────────────


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join("/tmp", f"tsk_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.fh.close()

    def summary(self):
        if self.proc is None or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * (max(sm) if sm else 1)]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if _isnum(r[3])), default=None)}


def _isnum(s):
    try:
        float(s)
        return True
    except ValueError:
        return False


# ── CPU side (reference arm / cpu_baseline): the oracle port ───────────────


ORACLE_PLANNERS = {
    "periodic": lambda orc, q, ix: orc.plan_periodic(q, S_BATCH, ix),
    "setsplit_fixed": lambda orc, q, ix: orc.plan_setsplit_fixed(q, ix, -(-orc.store_len(q) // S_BATCH)),
    "setsplit_max": lambda orc, q, ix: orc.plan_setsplit_max(q, ix, S_BATCH),
    "setsplit_minmax": lambda orc, q, ix: orc.plan_setsplit_minmax(q, ix, 16, S_BATCH),
    "greedy_min": lambda orc, q, ix: orc.plan_greedy(q, ix, S_BATCH, "min"),
    "greedy_max": lambda orc, q, ix: orc.plan_greedy(q, ix, S_BATCH, "max"),
}


def cpu_setup(e_cols, q_cols, presorted=False, planner="periodic", table=None):
    """Oracle store/index/plan for the reference algorithm (numpy port) plus an
    evenly spread batch order for sampling.  ``table`` reuses an existing
    plan's (lo, hi) batches instead of re-planning."""
    from oracle import oracle as orc

    t0 = time.perf_counter()
    e = orc.make_store(*(e_cols[k] for k in FIELDS), presorted=presorted)
    q = orc.make_store(*(q_cols[k] for k in FIELDS), presorted=presorted)
    ix = orc.index_build(e, M_BINS)
    if table is not None:
        plan = [(int(a), int(b), None, None, None, None) for a, b in zip(*table)]
    else:
        plan = ORACLE_PLANNERS[planner](orc, q, ix)
    log(f"[cpu] oracle store/index/plan in {time.perf_counter() - t0:.1f}s, {len(plan)} batches")
    order = _spread(len(plan))
    return e, q, ix, plan, order


def _spread(n):
    """Deterministic batch order that samples the plan evenly (0, n/2, n/4, 3n/4, ...)."""
    seen, out = set(), []
    step = n
    while step >= 1 and len(out) < n:
        for k in range(0, n, step):
            if k not in seen:
                seen.add(k)
                out.append(k)
        step //= 2
    return out + [k for k in range(n) if k not in seen]


def time_cpu_batches(e, q, ix, plan, d, batch_ids, workers):
    from oracle import oracle as orc

    t0 = time.perf_counter()
    _, st = orc.search(e, ix, q, plan, d, workers=workers, batch_ids=batch_ids)
    return st["interactions"], time.perf_counter() - t0, st["hits"]


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    e_cols, q_cols = workload_columns(cfg)
    e, q, ix, plan, order = cpu_setup(e_cols, q_cols, planner=args.planner)
    # one step = a bounded sample of batches (~budget seconds of CPU work)
    budget = float(os.environ.get("TSK_REF_STEP_S", "8"))
    cursor = 0
    step_ints, step_secs, step_batches = [], [], []

    def one_step():
        nonlocal cursor
        ints = secs = 0.0
        ids = []
        while secs < budget and len(ids) < len(order):
            k = order[cursor % len(order)]
            cursor += 1
            i, s, _ = time_cpu_batches(e, q, ix, plan, cfg["d"], [k], workers)
            ints += i
            secs += s
            ids.append(k)
        return ints, secs, ids

    for _ in range(args.warmup):
        one_step()
    for _ in range(args.steps):
        i, s, ids = one_step()
        step_ints.append(i)
        step_secs.append(s)
        step_batches.append(len(ids))
    value = sum(step_ints) / sum(step_secs)
    sample = (f"{sum(step_batches)} batch evaluations (of {len(plan)} Periodic s={S_BATCH} batches) over {args.steps} steps "
              f"(evenly spread), {int(sum(step_ints))} interactions")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(step_secs) / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ── GPU side (our arm) ──────────────────────────────────────────────────────


def run_ours(args, cfg):
    import paper_1405_7461_b200 as tsk
    from paper_1405_7461_b200 import _native
    from paper_1405_7461_b200.engine import search_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # TSK_BENCH_DEVICE pins every rank to one GPU (multi-rank smoke test on a
    # single-GPU box; the timing collectives then run over gloo)
    forced = os.environ.get("TSK_BENCH_DEVICE")
    if forced is not None:
        local = int(forced)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        if forced is None:
            tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            tdist.init_process_group("gloo")
        dist = tdist
    tsk.set_device(local)
    d = cfg["d"] if args.d is None else args.d

    t0 = time.perf_counter()
    e_cols, q_cols = workload_columns(cfg)
    store = tsk.SegmentStore.from_columns(e_cols, validate=False)
    queries = tsk.SegmentStore.from_columns(q_cols, validate=False)
    del e_cols, q_cols
    t_gen = time.perf_counter() - t0
    index = tsk.build_index(store, M_BINS)
    t_plan0 = time.perf_counter()
    plan = PLANNERS[args.planner](tsk, queries, index)
    t_plan = time.perf_counter() - t_plan0
    t_setup = time.perf_counter() - t0
    ints_all = np.array([b.interactions for b in plan.batches], dtype=np.int64)
    b0, b1 = shard_bounds(ints_all, world)[rank]
    mine = sub_plan(plan, b0, b1)
    log(f"[rank {rank}] {len(store)} entries, {len(queries)} queries, {len(plan.batches)} batches; "
        f"shard [{b0},{b1}); setup {t_setup:.1f}s (gen {t_gen:.1f}s)")

    # pinned host copy of this rank's query columns for the e2e leg
    if mine is not None:
        pq = tsk.SegmentStore(*(_native.pinned_copy(np.ascontiguousarray(getattr(mine.queries, k)))
                                for k in FIELDS), validate=False, presorted=True)
        e2e_plan = tsk.BatchPlan(pq, mine.batches)

    def barrier():
        if dist is not None:
            dist.barrier()

    def _reduce(x: float, op) -> float:
        if dist is None:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cpu" if forced is not None else "cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def allmax(x: float) -> float:
        return _reduce(x, dist.ReduceOp.MAX if dist else None)

    def allsum(x: float) -> float:
        return _reduce(x, dist.ReduceOp.SUM if dist else None)

    fp64 = _native.probe_fp64(local)
    fp64_peak = max(fp64.values())
    fp32_peak = _native.probe_fp32(local)

    # ── value: queries resident in HBM, hits left in HBM ──
    res = None
    if mine is not None:
        res = search_device(store, index, mine, d)  # uploads the queries once
    # clocks are sampled from the warm-up through the e2e loop (short timed
    # regions would otherwise fall between nvidia-smi samples)
    clk = ClockSampler(local).__enter__()
    t_clk = time.perf_counter()
    for _ in range(args.warmup):
        if mine is not None:
            res = search_device(store, index, mine, d, queries_resident=True)
    barrier()
    dev_ms, k1_ms, launches, work, hits, ovl, evals = 0.0, 0.0, 0, 0.0, 0, 0, 0
    w0 = time.perf_counter()
    for _ in range(args.steps):
        if mine is None:
            continue
        r = search_device(store, index, mine, d, queries_resident=True)
        dev_ms += r.device_ms
        k1_ms += r.k1_ms
        launches += r.launches
        evals += r.k1_evals
        o = int(r.per_batch[:, 2].sum())
        ovl += o
        hits += r.n
        work += W_DECIDE * o + W_HIT * r.n
    wall_s = time.perf_counter() - w0
    barrier()
    my_ints = int(ints_all[b0:b1].sum())
    t_dev = allmax(dev_ms / 1e3)
    total_ints = allsum(float(my_ints)) * args.steps
    value = total_ints / t_dev if t_dev > 0 else 0.0

    # ── e2e: public drop-in call, pinned host inputs, results to host ──
    # warm-up also fills the pinned result pool: like the timed loop, the
    # previous result stays alive during the next call (two blocks alternate)
    rs = None
    for _ in range(max(2, args.warmup)):
        if mine is not None:
            rs, _ = tsk.run_search(store, index, e2e_plan, d)
    barrier()
    e2e_s, h2d, d2h, e2e_hits = 0.0, 0, 0, 0
    for _ in range(args.steps):
        if mine is None:
            continue
        t1 = time.perf_counter()
        rs, st = tsk.run_search(store, index, e2e_plan, d)
        e2e_s += time.perf_counter() - t1
        h2d += len(pq) * (2 * 8 + 8 * 8) + len(mine.batches) * 16
        d2h += len(rs) * 48 + len(mine.batches) * 32
        e2e_hits += len(rs)
        assert st.interactions_computed == my_ints
    while time.perf_counter() - t_clk < 0.3:  # at least a few samples
        time.sleep(0.05)
    clk.__exit__(None, None, None)
    t_e2e = allmax(e2e_s)
    e2e_value = total_ints / t_e2e if t_e2e > 0 else 0.0
    total_hits = allsum(float(hits))  # every rank joins every collective

    # roofline of the dominant kernel (K1), this rank
    k1_s = k1_ms / 1e3
    achieved = work / k1_s / 1e12 if k1_s > 0 else 0.0
    peak = fp64_peak / 1e12
    # the kernel as implemented: FP32 pre-filter ops per evaluated pair
    # (3 FFMA + 3 FADD separation, 3 norm, 1 compare, and one 2-op threshold per
    # query shared by a lane's 4 candidates) vs the
    # measured FFMA rate
    f32_achieved = F32_OPS * evals / k1_s / 1e12 if k1_s > 0 else 0.0
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(prof):
        try:
            tj = json.load(open(prof))
            if tj.get("config") == args.config:
                traffic = tj.get("dram_bytes_per_launch")
        except (OSError, ValueError):
            pass

    cpu = None
    if world == 1 and not args.no_cpu_baseline and rank == 0:
        workers = os.cpu_count() or 1
        sorted_cols = lambda s: {k: getattr(s, k) for k in FIELDS}  # noqa: E731
        e, q, ix, oplan, order = cpu_setup(sorted_cols(store), sorted_cols(queries), presorted=True,
                                           table=plan.table())
        ints = secs = 0.0
        nbat = 0
        budget = float(os.environ.get("TSK_CPU_BASELINE_S", "20"))
        for k in order:
            i, s, _ = time_cpu_batches(e, q, ix, oplan, d, [k], workers)
            ints += i
            secs += s
            nbat += 1
            if secs >= budget:
                break
        cpu = {"value": ints / secs, "unit": UNIT, "cores": workers, "kind": "port",
               "sample": f"{nbat} of {len(oplan)} batches (evenly spread), {int(ints)} interactions, "
                         f"{secs:.1f}s; numpy port of the reference algorithm, workers={workers}"}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_dev / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference datagen stream; entry DB resident, replicated per GPU)",
            "config": {
                "workload": f"{args.config}: {cfg['desc']}", "entries": len(store),
                "queries": len(queries), "batches": len(plan.batches), "d": d, "s": S_BATCH,
                "planner": args.planner, "plan_s": t_plan,
                "m": M_BINS, "interactions_per_step": int(total_ints / args.steps),
                "hits_per_step": int(total_hits / args.steps),
                "l2": "inputs larger than L2 (entry SoA 141 B/segment resident in HBM)",
                "parallelism": f"dp{world} (contiguous interaction-balanced batch shards; no collective)",
            },
            "response_time_s": t_e2e / args.steps,
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d / args.steps),
                    "d2h_bytes_per_step": int(d2h / args.steps),
                    "call": "paper_1405_7461_b200.run_search(store, index, plan, d) (pinned host queries)"},
            "roofline": {
                "bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None, "traffic": traffic,
                "kernel": "k1_pairs", "work": f"{W_DECIDE}*overlapping pairs + {W_HIT}*hits FP64 flops",
                "k1_ms_per_step": k1_ms / args.steps,
                "peak_source": "tsk_probe_fp64 on this GPU in this run (DADD/DMUL/DFMA ops/s); "
                               "MEASURED_PEAKS.json has no FP64 figure",
                "hbm_bytes_per_step": None,
            },
            "kernel_roofline": {
                "bound": "fp32 issue (K1's FP32 pre-filter)", "kernel": "k1_pairs_f32",
                "work": f"{F32_OPS} FP32 ops per evaluated (candidate, query) pair",
                "evaluated_pairs_per_step": int(evals / args.steps),
                "achieved": f32_achieved, "peak": fp32_peak / 1e12, "unit": "TOP/s",
                "frac": f32_achieved * 1e12 / fp32_peak if fp32_peak else None,
                "peak_source": "tsk_probe_fp32 on this GPU in this run (FFMA ops/s, one op per FFMA)",
            },
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": launches,
            "wall_s_value_steps": wall_s,
            "setup_s": t_setup,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c5")
    ap.add_argument("--d", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--planner", choices=sorted(PLANNERS), default="periodic",
                    help="batch planner (config 4 compares them; PAPER.md Table 3)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
