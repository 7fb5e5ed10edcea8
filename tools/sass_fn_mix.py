"""Static opcode mix of one kernel in a `cuobjdump -sass` listing.
    python tools/sass_fn_mix.py listing.sass <mangled-name substring>"""
import collections
import re
import sys

path, key = sys.argv[1], sys.argv[2]
on = False
cnt = collections.Counter()
for ln in open(path):
    if "Function :" in ln:
        on = key in ln
        continue
    if not on:
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        t = m.group(2).strip()
        op = t.split()[1] if t.startswith("@") else t.split()[0]
        cnt[op.split(".")[0]] += 1
print(sum(cnt.values()), "instructions")
print("  ".join(f"{k}:{v}" for k, v in cnt.most_common(45)))
