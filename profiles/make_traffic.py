"""Write profiles/ncu_traffic.json (bench.py's roofline.traffic / roofline.l2)
from the raw page of an ncu --set full capture of the bench's PCG loop.

usage: python profiles/make_traffic.py raw.csv "<how it was captured>"
"""
import collections
import csv
import json
import os
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
col = {k: hdr.index(k) for k in ("Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum",
                                  "gpu__time_duration.sum", "lts__t_sectors.sum",
                                  "lts__t_sectors_srcunit_tex_op_read.sum")}
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "sector": 1.0, "Ksector": 1e3, "Msector": 1e6}
acc = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].replace("bdem::", "")
    t_us = float(r[col["gpu__time_duration.sum"]].replace(",", "")) * \
        scale.get(units[col["gpu__time_duration.sum"]], 1.0)
    if t_us < 6.0:       # launches that exited at once (the solve had stopped)
        continue
    for k, i in col.items():
        if k == "Kernel Name":
            continue
        acc[name][k].append(float(r[i].replace(",", "")) * scale.get(units[i], 1.0))
out = {}
for name, m in acc.items():
    n = len(m["gpu__time_duration.sum"])
    avg = {k: sum(v) / n for k, v in m.items()}
    out[name] = {"dram_bytes_per_launch": avg["dram__bytes_read.sum"] + avg["dram__bytes_write.sum"],
                 "ncu_time_us": avg["gpu__time_duration.sum"], "launches_captured": n,
                 "l2_sectors_per_launch": avg["lts__t_sectors.sum"],
                 "l2_tex_read_sectors_per_launch": avg["lts__t_sectors_srcunit_tex_op_read.sum"],
                 "source": sys.argv[2]}
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
