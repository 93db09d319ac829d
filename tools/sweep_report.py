"""Dev helper: the §8d sweep bench lines (tools/gpurun/r2_s3_sweeps.sh) as a
markdown table: python tools/sweep_report.py gpurun_out/sw > profiles/r2_sweeps_8d.md"""
import glob
import json
import os
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/sw"
rows = []
for f in sorted(glob.glob(os.path.join(d, "*.json"))):
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except (ValueError, IndexError):
        rows.append((os.path.basename(f), None))
        continue
    rows.append((os.path.basename(f), line))


def key(r):
    n, l = r
    if l is None:
        return ("z", n)
    c = l["config"]
    return (c["workload"][:4], c.get("planner", ""), c["d"], c["s"])


print("# SURVEY §8d workload coverage, round 2 final kernel (B200, one GPU)")
print()
print("`tools/gpurun/r2_s3_sweeps.sh`: `bench.py --steps 5 --warmup 3 --no-cpu-baseline` per row, parity on 48")
print("evenly spread batches against the oracle (every batch when the plan has fewer), SM clock in the last column.")
print("value = pair-evals/s of the device pipeline (queries resident); e2e = through `run_search` with pinned host")
print("queries, result columns copied to the host.")
print()
print("| workload | planner | d | s | batches | hits/step | hit fraction | K1 ms | device ms | response ms | value | e2e | parity (batches, mismatches) | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for n, l in sorted(rows, key=key):
    if l is None:
        print(f"| {n} | (no line) |||||||||||||")
        continue
    c, p = l["config"], l.get("parity") or {}
    w = c["workload"].split(":")[0]
    frac = c["hits_per_step"] / c["interactions_per_step"]
    print(f"| {w} | {c.get('planner', 'periodic')} | {c['d']:g} | {c['s']} | {c['batches']} | {c['hits_per_step']:,} | {frac:.2e} | "
          f"{l['roofline']['k1_ms_per_step']:.2f} | {l['ms_per_step']:.2f} | {l['response_time_s'] * 1e3:.2f} | "
          f"{l['value']:.3e} | {l['e2e']['value']:.3e} | {p.get('batches')}, {p.get('mismatches')} | {l['clocks']['sm_mhz']:.0f} |")
