"""Print the key memory/occupancy metrics of an ncu report (raw page).

usage: python profiles/summarize.py report.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "launch__occupancy_limit_registers"]


def summarize(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0]
        print(f"== {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"   {k:62s} {r[i]:>16s} {units[i]}")
        stalls = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(r[i] or 0))
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_") and
                  not h.endswith("not_issued")]
        stalls.sort(key=lambda x: -x[1])
        tot = sum(v for _, v in stalls) or 1.0
        print("   stalls: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in stalls[:5]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        summarize(p)
