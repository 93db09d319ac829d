"""Calibrate the perfmodel on this GPU and check its predictions (dev tool).

    python tools/perfmodel_demo.py [--config c3] [--out profiles/r1_perfmodel_c3.md]

1. calibrate_surfaces on the default grid up to the workload's largest
   candidate count, calibrate_host for the query-set size;
2. estimate_hit_rates with a pool sampled like the workload's queries;
3. predict the response time of Periodic plans for several s and measure
   run_search for the same plans (median of 5), so the table shows
   predicted vs measured and the recommended s.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (workload definitions)
import paper_1405_7461_b200 as tsk  # noqa: E402
from paper_1405_7461_b200 import perfmodel as pm  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    tsk.set_device(0)
    cfg = bench.CONFIGS[args.config]
    e_cols, q_cols = bench.workload_columns(cfg)
    store = tsk.SegmentStore.from_columns(e_cols, validate=False)
    queries = tsk.SegmentStore.from_columns(q_cols, validate=False)
    index = tsk.build_index(store, bench.M_BINS)
    d = cfg["d"]
    lines = [f"# perfmodel on B200: config {args.config} ({cfg['desc']}), d={d}\n"]

    t = time.perf_counter()
    s_axis = (30, 60, 120, 240, 480)
    c_max = max(b.candidates for b in tsk.periodic(queries, max(s_axis), index).batches)
    sf = pm.calibrate_surfaces(pm.default_grid(max(c_max, 32)), reps=3)
    t_sf = time.perf_counter() - t
    t = time.perf_counter()
    host = pm.calibrate_host(len(queries), [16, 64, 256, 1024, 4096], reps=3)
    t_host = time.perf_counter() - t
    t = time.perf_counter()
    prof = pm.estimate_hit_rates(store, index, queries, 120, d, num_epochs=20, seed=1)
    t_prof = time.perf_counter() - t
    lines.append(f"calibrate_surfaces (10x10 grid, c up to {c_max:,}): {t_sf:.1f} s, noisy points {sf.noisy_points}; "
                 f"calibrate_host: {t_host:.1f} s (offset {host.offset:.3g} s, scale {host.scale:.3g}, "
                 f"exponent {host.exponent:.3f}, {host.transfer_per_byte:.3g} s/B); "
                 f"estimate_hit_rates: {t_prof:.2f} s, {prof.trials} rounds, converged={prof.converged}, "
                 f"global rate {prof.global_rate:.3g}\n")
    lines.append("| s | batches | predict s | predicted kernel ms | predicted host ms | predicted total ms | "
                 "measured run_search ms (median of 5) | measured device ms |")
    lines.append("|---|---|---|---|---|---|---|---|")
    best, preds = pm.recommend_batch_size(s_axis, queries, store, index, sf, prof, host, d)
    for p in preds:
        t = time.perf_counter()
        pm.predict(p.s, queries, store, index, sf, prof, host, d)
        t_pred = time.perf_counter() - t
        plan = tsk.periodic(queries, p.s, index)
        tsk.run_search(store, index, plan, d)
        meas, dev = [], []
        for _ in range(5):
            t = time.perf_counter()
            _, st = tsk.run_search(store, index, plan, d)
            meas.append(time.perf_counter() - t)
            dev.append(st.device_seconds)
        lines.append(f"| {p.s} | {len(plan.batches)} | {t_pred:.3f} | {p.kernel_seconds * 1e3:.2f} | "
                     f"{p.host_seconds * 1e3:.2f} | {p.total_seconds * 1e3:.2f} | {np.median(meas) * 1e3:.2f} | "
                     f"{np.median(dev) * 1e3:.2f} |")
    lines.append(f"\nrecommend_batch_size → s = {best}")
    text = "\n".join(lines) + "\n"
    print(text)
    if args.out:
        open(args.out, "w").write(text)


if __name__ == "__main__":
    main()
