"""Summarise an `ncu --page source --csv --print-source sass` export: warp
instructions and stall samples per opcode, plus the hottest instructions.
Only the first kernel in the export is read."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ie = h.index("Instructions Executed")
sm = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= max(sm, ie) or not r[ie].isdigit():
        if data:
            break
        continue
    data.append(r)
op, st = collections.Counter(), collections.Counter()
tot = tots = 0
for r in data:
    t = r[1].split()
    o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
    n, s = int(r[ie]), int(r[sm] or 0)
    op[o] += n
    st[o] += s
    tot += n
    tots += s
print("total warp inst", tot, "samples", tots)
for o, n in op.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{o:10s} {n:10d} {100*n/tot:5.1f}%  stall {100*st[o]/max(tots,1):5.1f}%")
print()
for r in sorted(data, key=lambda r: -int(r[sm] or 0))[:30]:
    print(r[sm], r[ie], r[0][-5:], r[1][:80])
