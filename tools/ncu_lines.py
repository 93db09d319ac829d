"""Dev helper: per-source-line stall samples and instructions of an ncu report
(ncu --page source --print-source cuda,sass), top N lines."""
import csv, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fn, rows, tot_s, tot_i = None, [], 0, 0
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fn = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No") or r[0] == "":
        continue
    try:
        s, i = int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    rows.append((s, i, f"{fn}:{r[0]}", r[1].strip()[:90]))
    tot_s += s
    tot_i += i
rows.sort(reverse=True)
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, loc, src in rows[:top]:
    print(f"{100*s/tot_s:5.1f}% smp {100*i/max(tot_i,1):5.1f}% ins  {loc:22s} {src}")
