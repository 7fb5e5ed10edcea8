"""Opcode mix of the grid kernel's chunk loops in a SASS listing: every
backward-branch loop that contains MUFU ops, divided by the cells one
iteration computes (4 per lane).  Branch-skipped blocks (the partial-chunk
store path) are counted too, so this is an upper bound for full chunks."""
import collections
import re
import sys

CELLS_PER_LANE = 4
PACKED = ("FFMA2", "FMUL2", "FADD2")
ins = []
for ln in open(sys.argv[1]):
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
# innermost loops only (no other loop nested inside)
inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
for i0, i1 in inner:
    cnt = collections.Counter()
    for _, txt in ins[i0:i1 + 1]:
        op = txt.split()[1] if txt.startswith("@") else txt.split()[0]
        cnt[op.split(".")[0]] += 1
    if not cnt["MUFU"]:
        continue
    n = i1 - i0 + 1
    fp32 = sum(v * (2 if k in PACKED else 1) for k, v in cnt.items()
               if k in PACKED + ("FFMA", "FMUL", "FADD"))
    print(f"loop @{ins[i0][0]:#x}: {n} instr ({n / CELLS_PER_LANE:.1f}/cell), "
          f"fp32 lane-ops {fp32 / CELLS_PER_LANE:.1f}/cell, MUFU {cnt['MUFU'] / CELLS_PER_LANE:.2f}/cell")
    print("   " + "  ".join(f"{k}:{v / CELLS_PER_LANE:.2f}" for k, v in cnt.most_common(18)))
