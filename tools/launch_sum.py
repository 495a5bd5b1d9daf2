"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).

    python tools/launch_sum.py launches.csv [skip_first_n]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ix = {k: j for j, k in enumerate(hdr)}
tot, cnt = defaultdict(float), defaultdict(int)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
for r in rows[h + 1:]:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0][:70]
    tot[name] += float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    cnt[name] += 1
all_ = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("%10.1f us %5.1f%% %4d  %s" % (v, 100 * v / all_, cnt[k], k))
