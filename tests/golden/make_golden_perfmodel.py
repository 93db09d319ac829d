"""Golden vectors for the perfmodel drop-in, produced by the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_perfmodel.py

Writes tests/golden/perfmodel.npz and tests/golden/perfmodel_doc.txt from
trajseek.perfmodel (/root/reference/pkg/src/trajseek/perfmodel.py):

  fit_*        fit_power_law on noiseless, noisy, constant and offset
               samples (perfmodel.py:72-128)
  lk_*         BenchSurfaces.lookup on a synthetic grid (perfmodel.py:398-451)
  hr*_*        estimate_hit_rates on two generated scenes (perfmodel.py:199-299)
  tm_*         temporal_miss_fraction of every Periodic batch (perfmodel.py:327-343)
  mix_*        interaction_mix of every batch (perfmodel.py:346-364)
  pred_*       predict / recommend_batch_size (perfmodel.py:656-731)
  perfmodel_doc.txt  save_model of a full model (perfmodel.py:749-783)

The scenes come from datagen profiles that this package reproduces byte for
byte (tests/golden/datagen.npz), so the tests rebuild them locally.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
HERE = os.path.dirname(os.path.abspath(__file__))

from trajseek import build_index, datagen, perfmodel  # noqa: E402  (the reference)
from trajseek.planner import periodic  # noqa: E402

# scenes: (store profile, m, pool profile, queries sample, d, s, epochs, seed)
SCENES = {
    "small": (("uniform", 6, 3, 150), 60, ("uniform", 6, 8, 150), (2, 11), 20.0, 10, 8, 0),
    "c1": (("uniform", 200, 1, 100), 200, ("uniform", 100, 2, 100), (10, 3), 5.0, 20, 10, 5),
}


def scene(name):
    (k, n, seed, ts), m, (pk, pn, pseed, pts), (nq, qseed), d, s, ne, rseed = SCENES[name]
    store = datagen.generate(datagen.make_profile(k, n, seed=seed, timesteps=ts))
    index = build_index(store, m)
    pool = datagen.generate(datagen.make_profile(pk, pn, seed=pseed, timesteps=pts))
    queries = datagen.sample_queries(pool, nq, seed=qseed)
    return store, index, pool, queries, d, s, ne, rseed


def synthetic_surfaces(c_max):
    grid = perfmodel.default_grid(c_max)
    rng = np.random.default_rng(77)
    shape = (len(grid.q_axis), len(grid.c_axis))
    q = np.asarray(grid.q_axis, dtype=np.float64)[:, None]
    c = np.asarray(grid.c_axis, dtype=np.float64)[None, :]
    base = 2e-5 + 1e-9 * q * c
    grids = [base * (1.5 + 0.3 * rng.random(shape)), base * (0.2 + 0.05 * rng.random(shape)),
             base * (1.0 + 0.2 * rng.random(shape)), np.full(shape, 1e-5) + 1e-7 * rng.random(shape)]
    return perfmodel.BenchSurfaces(q[:, 0].copy(), c[0].copy(), *grids, 3)


def main():
    out = {}
    # power-law fits
    rng = np.random.default_rng(5)
    s = np.array([1, 2, 4, 8, 16, 32, 64, 128], dtype=np.float64)
    cases = [
        (s, 0.002 + 0.03 * s**-0.6),
        (s, -0.001 + 0.5 * s**-1.3),
        (s, 1e-4 + 2e-3 * s**0.7),
        (s, (0.004 + 0.02 * s**-0.8) * (1 + 0.02 * rng.standard_normal(s.shape[0]))),
        (s[:5], np.full(5, 0.25)),
        (np.array([3.0, 7.0, 11.0, 30.0]), np.array([0.9, 0.41, 0.33, 0.2])),
    ]
    for k, (x, y) in enumerate(cases):
        f = perfmodel.fit_power_law(x, y)
        out[f"fit{k}_s"], out[f"fit{k}_t"] = x, y
        out[f"fit{k}_out"] = np.array([f.offset, f.scale, f.exponent, f.rss, float(f.degenerate)])

    # surface lookups
    sf = synthetic_surfaces(5000)
    out["sf_q"], out["sf_c"] = sf.q_axis, sf.c_axis
    for name in ("all_hit", "temporal_miss", "spatial_miss", "launch"):
        out[f"sf_{name}"] = getattr(sf, name)
    pts_i = np.concatenate([rng.uniform(0, 400 * 6000, 300), [0.0, 16.0, 300 * 5000.0]])
    pts_c = np.concatenate([rng.uniform(1, 6000, 300), [16.0, 16.0, 5000.0]])
    out["lk_i"], out["lk_c"] = pts_i, pts_c
    for name in ("all_hit", "temporal_miss", "spatial_miss", "launch"):
        out[f"lk_{name}"] = np.array([sf.lookup(name, a, b) for a, b in zip(pts_i, pts_c)])

    host = perfmodel.HostOverheadModel(1000, 1e-3, 5e-3, -0.7, 1e-9)
    hosts = (host, perfmodel.HostOverheadModel(10, 2e-4, 1e-3, -0.5, 2e-9))
    for name in SCENES:
        store, index, pool, queries, d, sb, ne, rseed = scene(name)
        prof = perfmodel.estimate_hit_rates(store, index, pool, sb, d, num_epochs=ne, seed=rseed)
        out[f"hr_{name}_rates"] = np.array([e.rate for e in prof.epochs])
        out[f"hr_{name}_sampled"] = np.array([e.sampled for e in prof.epochs])
        out[f"hr_{name}_bounds"] = np.array([[e.interval.begin, e.interval.end] for e in prof.epochs])
        out[f"hr_{name}_meta"] = np.array([prof.t0, prof.t_max, prof.d, prof.sample_batch_size,
                                           prof.global_rate, prof.trials, float(prof.converged)])
        plan = periodic(queries, sb, index)
        tm, mix = [], []
        for b in plan.batches:
            if b.first is None:
                continue
            batch = queries.view(b.lo, b.hi)
            tm.append(perfmodel.temporal_miss_fraction(store, (b.first, b.last), batch))
            m = perfmodel.interaction_mix(store, (b.first, b.last), batch, prof)
            mix.append([m.hit, m.temporal_miss, m.spatial_miss, float(m.clamped)])
        out[f"tm_{name}"] = np.array(tm)
        out[f"mix_{name}"] = np.array(mix)
        preds = []
        for sv in (3, 5, 10, 20, 40):
            p = perfmodel.predict(sv, queries, store, index, sf, prof, host, d)
            preds.append([p.s, p.host_seconds, p.kernel_seconds, p.total_seconds, p.result_bytes,
                          p.predicted_hits, p.clamped_batches])
        out[f"pred_{name}"] = np.array(preds)
        best, _ = perfmodel.recommend_batch_size([40, 3, 10, 5, 20], queries, store, index, sf, prof, host, d)
        out[f"rec_{name}"] = np.array([best])
        if name == "c1":
            perfmodel.save_model(perfmodel.PerfModel(sf, prof, hosts), os.path.join(HERE, "perfmodel_doc.txt"))
    np.savez_compressed(os.path.join(HERE, "perfmodel.npz"), **out)
    print("wrote perfmodel.npz,", len(out), "arrays; perfmodel_doc.txt")


if __name__ == "__main__":
    main()
