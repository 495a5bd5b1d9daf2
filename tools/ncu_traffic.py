"""DRAM traffic per launch of each kernel in an `ncu --set full` report, written
to profiles/traffic.json for bench.py's roofline "traffic" field.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep cfg5_allen_cahn_scaleout [source-label] [profiles/traffic.json]

Entries of other kernels already in the file for the workload are kept; `source-label`
(default: the report's file name) names the committed summary of the capture.
"""
import csv
import io
import json
import os
import re
import subprocess
import sys


def main(rep, workload, label=None, out="profiles/traffic.json"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    res = {}
    for d in data:
        name = d[idx["Kernel Name"]]
        m = re.search(r"k_(\w+?)_tc", name)
        key = "bsde_" + (m.group(1) if m else name)
        tot = 0.0
        for met in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = idx[met]
            tot += float(d[i].replace(",", "")) * scale.get(units[i], 1)
        res.setdefault(key, []).append(tot)
    db = json.load(open(out)) if os.path.exists(out) else {}
    entry = db.setdefault(workload, {})
    for k, v in res.items():
        entry[k] = {"bytes_per_launch": sum(v) / len(v), "source": label or os.path.basename(rep)}
    json.dump(db, open(out, "w"), indent=1)
    print(json.dumps(db[workload], indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
