"""Dev helper: list the innermost backward-branch loops of a kernel's SASS
that contain FP64 compares (K1's pair loops) with their instruction mix."""
import re, subprocess, sys
from collections import Counter

obj, kern = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "k1_pairs")
out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0]
    if kern not in name or "rare_flush" in name:
        continue
    ins = []
    for line in f.split("\n"):
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr_idx = {a: i for i, (a, _) in enumerate(ins)}
    for i, (a, txt) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)\s*)?(0x[0-9a-f]+)", txt)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= a or tgt not in addr_idx:
            continue
        body = ins[addr_idx[tgt]: i + 1]
        if not any("DSETP" in t for _, t in body) or len(body) > 400:
            continue
        ops = Counter(t.split()[0] if not t.startswith("@") else t.split()[1] for _, t in body)
        fp64 = sum(v for k, v in ops.items() if k.split(".")[0] in ("DADD", "DMUL", "DFMA", "DSETP"))
        print(f"loop {tgt:#x}-{a:#x}: {len(body)} instr, FP64 {fp64}, other {len(body) - fp64}")
        print("   ", ", ".join(f"{k}:{v}" for k, v in ops.most_common() if k.split('.')[0] not in ("DADD", "DMUL", "DFMA")))
