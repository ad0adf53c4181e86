"""Write profiles/ncu_traffic.json (bench.py's roofline.traffic / l2, assembly
traffic and FP64 fractions, C5 FP64 roofline) from the round-2 captures:

  prof_pcg_r02.ncu-rep    ncu --set full of the in-chain PCG kernels (600K plate)
  plate_asm_fp64.csv      ncu --metrics of k_bond_rows / k_element_assemble (600K plate)
  c5_asm_fp64.csv         the same for the C5 2M block, random q (k_bond_rows, k_bond_clamp)

usage: python profiles/make_traffic_r02.py <dir with the three files>
(scratch/r02/prof_r02.sh made them on a B200)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

d = sys.argv[1]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0,
         "msecond": 1e3, "sector": 1.0, "Ksector": 1e3, "Msector": 1e6, "inst": 1.0,
         "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "%": 1.0, "register/thread": 1.0,
         "ns": 1e-3, "us": 1.0, "ms": 1e3}


def pcg_kernels():
    out = subprocess.run(["ncu", "-i", os.path.join(d, "prof_pcg_r02.ncu-rep"), "--page", "raw",
                          "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    keys = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "lts__t_sectors.sum", "lts__t_sectors_srcunit_tex_op_read.sum")
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("bdem::", "")
        for k in keys:
            i = hdr.index(k)
            acc[name][k].append(float(r[i].replace(",", "")) * SCALE.get(units[i], 1.0))
    res = {}
    for name, m in acc.items():
        n = len(m["gpu__time_duration.sum"])
        a = {k: sum(v) / n for k, v in m.items()}
        res[name] = {"dram_bytes_per_launch": a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"],
                     "ncu_time_us": a["gpu__time_duration.sum"], "launches_captured": n,
                     "l2_sectors_per_launch": a["lts__t_sectors.sum"],
                     "l2_tex_read_sectors_per_launch": a["lts__t_sectors_srcunit_tex_op_read.sum"],
                     "source": "ncu --set full --cache-control none --clock-control none of the "
                               "PCG kernels inside bdem_pcg_iterate chains on the 600K plate "
                               "system (scratch/pcg_micro.py, scratch/r02/prof_r02.sh; "
                               "profiles/r02/prof_pcg_r02_*)"}
    return res


def metric_csv(path, what):
    rows = [r for r in csv.reader(open(path)) if len(r) > 12 and r[0] != "ID"]
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        name = r[4].split("(")[0]
        acc[(name, r[0])][r[12]] = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
    per = collections.defaultdict(list)
    for (name, _), m in acc.items():
        per[name].append(m)
    res = {}
    for name, ms in per.items():
        a = {k: sum(m[k] for m in ms) / len(ms) for k in ms[0]}
        flops = (2 * a["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"]
                 + a["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]
                 + a["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"])
        res[name] = {"dram_bytes_per_launch": a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"],
                     "ncu_time_us": a["gpu__time_duration.sum"], "launches_captured": len(ms),
                     "fp64_flops_per_launch": flops,
                     "fp64_pipe_frac":
                         a["sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"] / 100,
                     "registers": a["launch__registers_per_thread"],
                     "warps_active_frac":
                         a["sm__warps_active.avg.pct_of_peak_sustained_active"] / 100,
                     "source": f"ncu --metrics (scratch/r02/prof_r02.sh), {what}"}
    return res


out = pcg_kernels()
out.update(metric_csv(os.path.join(d, "plate_asm_fp64.csv"),
                      "600K plate step-1 predictor (scratch/r02/asm_once.py)"))
out["c5_block"] = metric_csv(os.path.join(d, "c5_asm_fp64.csv"),
                             "C5 2M block random q (scratch/r02/c5_once.py)")
path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
