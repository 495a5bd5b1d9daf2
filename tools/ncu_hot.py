"""Hottest SASS instructions of an ncu source page (csv): samples and top stall reasons.

    ncu -i rep --page source --csv > src.csv;  python tools/ncu_hot.py src.csv [N]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h0 = next(i for i, r in enumerate(rows) if "Source" in r and "Address" in r)
hdr = rows[h0]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[h0 + 1:] if len(r) == len(hdr) and r[0] != "Address"]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
byop = Counter()
reason = Counter()
for r in data:
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    byop[op.split(".")[0]] += n
    for st in stalls:
        reason[st] += int(r[ix[st]] or 0)
print("total samples", tot)
print("by reason:", ", ".join("%s %.1f%%" % (k[6:], 100.0 * v / tot) for k, v in reason.most_common(10)))
print("by opcode:", ", ".join("%s %.1f%%" % (k, 100.0 * v / tot) for k, v in byop.most_common(20)))
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
top = sorted(range(len(data)), key=lambda i: -int(data[i][ix["Warp Stall Sampling (All Samples)"]] or 0))[:N]
for i in sorted(top):
    r = data[i]
    n = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    rs = sorted(((int(r[ix[st]] or 0), st[6:]) for st in stalls), reverse=True)[:3]
    print("%5d %5.2f%% %-60s %s" % (i, 100.0 * n / tot, r[ix["Source"]][:60], " ".join("%s:%d" % (b, a) for a, b in rs if a)))
