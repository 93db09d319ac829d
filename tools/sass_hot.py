"""Dev helper: print the common path of each K1 pair loop (from the loop head
to the first VOTE-guarded branch, plus the loop tail), non-FP64 ops only."""
import re, subprocess, sys
obj = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
ins, f = [], False
for line in out.split("\n"):
    if "Function :" in line:
        f = "k1_pairs" in line and "rare" not in line
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if f and m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
idx = {a: i for i, (a, _) in enumerate(ins)}
FP = ("DADD", "DMUL", "DFMA", "FADD", "FMUL", "FFMA")
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\s+(0x[0-9a-f]+)", t)
    if not m or int(m.group(1), 16) >= a or int(m.group(1), 16) not in idx:
        continue
    h = idx[int(m.group(1), 16)]
    body = ins[h:i + 1]
    nfp = sum(1 for _, x in body if x.split()[0].split(".")[0] in FP)
    if nfp < 20:
        continue
    # common path = head .. first "@!P BRA" after a VOTE
    k = next((j for j, (_, x) in enumerate(body) if x.startswith("VOTE.ANY")), None)
    common = body[:k + 2] if k is not None else body
    tail = body[-4:]
    c_fp = sum(1 for _, x in common if x.split()[0].split(".")[0] in FP)
    other = [x for _, x in common if x.split()[0].split(".")[0] not in FP]
    print(f"loop {ins[h][0]:#x}: common {len(common)} instr ({c_fp} FP adds/muls/fmas), other: {'; '.join(o.split(' ')[0] for o in other)} | tail: {'; '.join(x for _, x in tail)}")
