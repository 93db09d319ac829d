"""Dev helper: turn a gpurun evidence directory into profiles/ summaries."""
import csv, glob, json, os, re, subprocess, sys
from collections import defaultdict

ev = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ev4"
P = "profiles"
summ = subprocess.run([sys.executable, "tools/ncu_summary.py", f"{ev}/k1_c5.ncu-rep"], capture_output=True, text=True).stdout
open(f"{P}/r1_k1_c5_final_ncu_full.txt", "w").write(summ)
rows = list(csv.reader(open(f"{ev}/launches_c5.csv")))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) > vi:
        n = r[ki].split("(")[0][:70]
        agg[n][0] += 1
        agg[n][1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
with open(f"{P}/r1_launches_c5_final.txt", "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 1 --warmup 1 --no-cpu-baseline\n")
    f.write("# config c5 (1e8 entries, 400k queries, d=1), final round-1 kernel; ns; cold-cache serialised: compare shares\n")
    f.write(f"{'kernel':72s} {'launches':>8s} {'total_ns':>14s} {'share':>7s}\n")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{n:72s} {c:8d} {t:14.0f} {t / tot * 100:6.2f}%\n")
rd = float(re.search(r"dram__bytes_read.sum\s+([\d.]+) Gbyte", summ).group(1)) * 1e9
wm = re.search(r"dram__bytes_write.sum\s+([\d.]+) (\w+)", summ)
wr = float(wm.group(1)) * (1e9 if wm.group(2) == "Gbyte" else 1e6)
json.dump({"config": "c5", "kernel": "k1_pairs_f32", "dram_bytes_per_launch": int(rd + wr),
           "source": "ncu --set full capture, profiles/r1_k1_c5_final_ncu_full.txt"},
          open(f"{P}/k1_traffic.json", "w"), indent=1)
for c in ("c1", "c2", "c3", "c4", "c5"):
    os.replace(f"{ev}/bench_{c}.json", f"{P}/r1_bench_{c}.json") if os.path.exists(f"{ev}/bench_{c}.json") else None
if os.path.exists(f"{ev}/bench_c3_2rank_samegpu.json"):
    os.replace(f"{ev}/bench_c3_2rank_samegpu.json", f"{P}/r1_bench_c3_2rank_samegpu.json")
# d sweep
with open(f"{P}/r1_dsweep_c3.md", "w") as f:
    f.write("# Config 3 d-sweep (RandWalk-Normal 1e7 entries x 40k queries, Periodic s=120, m=10,000), B200, round 1\n\n")
    f.write("| d | hits/step | device ms | K1 ms | response ms (e2e) | value pair-evals/s | e2e pair-evals/s | K1 frac |\n|---|---|---|---|---|---|---|---|\n")
    for d in (1, 5, 15, 30, 50):
        x = json.loads(open(f"gpurun_out/ds/c3_d{d}.json").read().strip().splitlines()[-1])
        f.write(f"| {d} | {x['config']['hits_per_step']:,} | {x['ms_per_step']:.2f} | {x['roofline']['k1_ms_per_step']:.2f} | "
                f"{x['response_time_s'] * 1e3:.2f} | {x['value']:.3e} | {x['e2e']['value']:.3e} | {x['roofline']['frac']:.3f} |\n")
    f.write("\nLarge d: each hit is re-evaluated exactly and solved (sqrt + 2 IEEE divisions) in queued, converged batches of 32; "
            "e2e at d >= 30 is dominated by the D2H of 48 B/hit result columns (15 GB at d = 50, ~57 GB/s).\n")
# planners
rows = []
for fpath in sorted(glob.glob("gpurun_out/pl/c4_*.json")):
    d = json.loads(open(fpath).read().strip().splitlines()[-1])
    c = d["config"]
    rows.append((c["planner"], c["batches"], c["plan_s"], c["interactions_per_step"], d["ms_per_step"], d["value"], d["e2e"]["value"], c["entries"]))
with open(f"{P}/r1_planners_c4.md", "w") as f:
    f.write("# Config 4 planner comparison (round 1, B200, final K1)\n\n")
    f.write(f"Workload c4: RandWalk-Exp 140,000 trajectories ({rows[0][7]:,} entry segments), 1,000 query trajectories, d=5, m=10,000; "
            "planner settings of PAPER.md Table 3 at s=120: SetSplit-Fixed(ceil(n/120)), SetSplit-Max(120), SetSplit-MinMax(16,120), Greedy-Min/Max(120).\n")
    f.write("`plan_s` = native C++ planner on the GPU box's host; device ms = search pipeline with queries resident (bench `value` leg).\n\n")
    f.write("| planner | batches | plan_s | interactions | device ms | value pair-evals/s | e2e pair-evals/s |\n|---|---|---|---|---|---|---|\n")
    for r in sorted(rows, key=lambda r: r[4]):
        f.write(f"| {r[0]} | {r[1]} | {r[2]:.3f} | {r[3]:,} | {r[4]:.2f} | {r[5]:.3e} | {r[6]:.3e} |\n")
    f.write("\nDevice time varies little across planners: K1 skips temporally disjoint (query, candidate) pairs per warp by bisection, so the "
            "extra interactions of a coarser plan cost almost nothing; overlapping pairs are plan-invariant.  The reference reports a 3.4% spread "
            "(PAPER.md:1239-1257).\n")
print(summ)
