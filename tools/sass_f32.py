"""Dev helper: common-path instruction counts of k1_pairs_f32's inner loops."""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
ins, f = [], False
for line in out.split("\n"):
    if "Function :" in line:
        f = "k1_pairs_f32" in line
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if f and m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
idx = {a: i for i, (a, _) in enumerate(ins)}
FP = ("FADD", "FMUL", "FFMA", "FFMA2", "FADD2", "FMUL2")
for i, (a, t) in enumerate(ins):
    m = re.search(r"BRA\s+(0x[0-9a-f]+)", t)
    if not m:
        continue
    tg = int(m.group(1), 16)
    if tg >= a or tg not in idx:
        continue
    body = ins[idx[tg]:i + 1]
    if sum(1 for _, x in body if x.split()[0].split(".")[0] in FP) < 30:
        continue
    k = next((j for j, (_, x) in enumerate(body) if x.startswith("VOTE.ANY")), None)
    common = body[:k + 2] if k is not None else body
    nfp = sum(1 for _, x in common if x.split()[0].split(".")[0] in FP)
    other = [x.split()[0] for _, x in common if x.split()[0].split(".")[0] not in FP]
    print(hex(ins[idx[tg]][0]), "common", len(common), "fp", nfp, other)
