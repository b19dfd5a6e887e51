"""Merge the DRAM traffic of one decode launch's attend kernels (an ncu --set
full capture) into profiles/traffic.json under key CONFIG/BITS; bench.py reads
it for roofline.traffic.
usage: traffic_from_ncu.py REPORT CONFIG BITS KERNEL_REGEX [KERNEL_REGEX ...]
(one launch of each named kernel: the first match in the report)."""
import csv
import json
import os
import re
import subprocess
import sys

rep, config, bits, pats = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4:]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base",
                      "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
per = {}
for p in pats:
    for r in rows[2:]:
        if re.search(p, r[ik]):
            per[r[ik]] = int(float(r[ir])) + int(float(r[iw]))
            break
    else:
        raise SystemExit(f"no kernel matching {p} in {rep}")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "traffic.json")
tj = {}
if os.path.exists(path):
    tj = json.load(open(path))
if "configs" not in tj:
    tj = {"configs": {}, "note": "dram__bytes_read.sum + dram__bytes_write.sum of one decode "
                                  "launch's attend kernels (ncu --set full), per CONFIG/BITS"}
tj["configs"][f"{config}/{bits}"] = {"dram_bytes_per_launch": sum(per.values()),
                                     "per_kernel": per, "source": os.path.basename(rep)}
json.dump(tj, open(path, "w"), indent=1)
print(json.dumps(tj["configs"][f"{config}/{bits}"]))
