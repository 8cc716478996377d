"""Aggregate an `ncu --page source --csv --print-source cuda,sass` export per
CUDA source line: warp instructions executed and stall samples (top lines)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ins, smp, text = collections.Counter(), collections.Counter(), {}
f = None
hdr = None
line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= max(ie, sm):
        continue
    if r[0].strip():
        line = (f, int(r[0]))
        text[line] = r[1].strip()[:90]
    if r[2].strip() and line is not None:
        try:
            ins[line] += int(r[ie] or 0)
            smp[line] += int(r[sm] or 0)
        except ValueError:
            pass
ti, ts = sum(ins.values()), sum(smp.values())
print(f"total warp inst {ti}  samples {ts}")
for k, v in ins.most_common(top):
    print(f"{100 * v / ti:5.1f}% inst {100 * smp[k] / max(ts, 1):5.1f}% stall  {k[0]}:{k[1]}  {text.get(k, '')}")
