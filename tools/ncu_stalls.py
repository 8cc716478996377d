"""Stall/opcode breakdown of one kernel from an `ncu --set full` capture:
  python tools/ncu_stalls.py REP.ncu-rep KERNEL_REGEX [TOP]"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
if kre != "all":
    cmd += ["-k", f"regex:{kre}"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ie = hdr.index("Instructions Executed")
sm = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
sidx = [hdr.index(h) for h in stalls]
tot, opc, opcs = collections.Counter(), collections.Counter(), collections.Counter()
T = S = 0
lines = []
for r in rows[2:]:
    if len(r) <= max(sm, ie) or not r[ie]:
        continue
    try:
        n, s = int(r[ie]), int(r[sm] or 0)
    except ValueError:
        continue
    T += n
    S += s
    toks = r[1].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]).split(".")[0]
    opc[op] += n
    opcs[op] += s
    st = {}
    for h, i in zip(stalls, sidx):
        try:
            v = int(r[i] or 0)
        except ValueError:
            v = 0
        tot[h] += v
        if v:
            st[h[6:]] = v
    lines.append((s, r[0], r[1][:60], n, sorted(st.items(), key=lambda x: -x[1])[:3]))
print(f"warp inst {T}  stall samples {S}")
for k, v in tot.most_common(10):
    print(f"  {k:28s} {100 * v / max(S, 1):5.1f}%")
for k, v in opc.most_common(top):
    print(f"  {k:10s} inst {100 * v / max(T, 1):5.1f}%  stall {100 * opcs[k] / max(S, 1):5.1f}%")
lines.sort(key=lambda x: -x[0])
for l in lines[:top]:
    print(" ", l[0], l[1], l[2], l[3], l[4])
