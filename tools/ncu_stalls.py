"""Dev helper: long-scoreboard (and other) stall samples per source line of
an ncu report (cuda,sass view), attributing each SASS row to its line."""
import csv, subprocess, sys, collections
rep, reason = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "stall_long_sb")
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ci = hdr.index(reason)
fn = line = None
agg, tot = collections.Counter(), 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        line = f"{fn}:{r[0]} {r[1].strip()[:70]}"
        continue
    try:
        v = int(r[ci])
    except (ValueError, IndexError):
        continue
    agg[line] += v
    tot += v
print(reason, "total", tot)
for k, v in agg.most_common(top):
    print(f"{100 * v / max(tot, 1):5.1f}% {k}")
