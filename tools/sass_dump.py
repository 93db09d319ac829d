"""Dev helper: dump the SASS of k1_pairs<true> between two addresses."""
import re, subprocess, sys
obj, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
kern = sys.argv[4] if len(sys.argv) > 4 else "k1_pairsILb1"
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
f = False
for line in out.split("\n"):
    if "Function :" in line:
        f = kern in line
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if f and m and lo <= int(m.group(1), 16) <= hi:
        print(m.group(1), m.group(2))
