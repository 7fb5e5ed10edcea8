"""Opcode mix of every innermost backward-branch loop of one kernel in a
`cuobjdump -sass` listing (static counts per loop iteration, all paths).
    python tools/sass_loops.py listing.sass <mangled-name substring>"""
import collections
import re
import sys

path, key = sys.argv[1], sys.argv[2]
on = False
ins = []
for ln in open(path):
    if "Function :" in ln:
        on = key in ln
        continue
    if on:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
idx = {a: i for i, (a, _) in enumerate(ins)}
loops = []
for i, (a, txt) in enumerate(ins):
    if "BRA" not in txt:
        continue
    m = re.search(r"0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < a and int(m.group(1), 16) in idx:
        loops.append((idx[int(m.group(1), 16)], i))
inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "FRND", "DMNMX")
for i0, i1 in sorted(inner):
    cnt = collections.Counter()
    for _, txt in ins[i0:i1 + 1]:
        op = txt.split()[1] if txt.startswith("@") else txt.split()[0]
        cnt[op.split(".")[0]] += 1
    n = i1 - i0 + 1
    f64 = sum(v for k, v in cnt.items() if k in FP64)
    print(f"loop @{ins[i0][0]:#x}-{ins[i1][0]:#x}: {n} instr, fp64-pipe {f64}, MUFU {cnt['MUFU']}")
    print("   " + "  ".join(f"{k}:{v}" for k, v in cnt.most_common(22)))
