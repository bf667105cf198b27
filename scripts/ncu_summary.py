"""Summarise an ncu report (raw page) for the kernels it holds."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__grid_size",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_red_lookup_miss.sum"]
def f(x):
    try: return float(x)
    except: return 0.0
for r in rows[2:]:
    print("----")
    for k in keys:
        if k in hdr:
            i = hdr.index(k); print(f"  {k} = {r[i]} {units[i]}")
    st = sorted(((f(r[i]), hdr[i]) for i in range(len(hdr)) if hdr[i].startswith("smsp__pcsamp_warps_issue_stalled") and not hdr[i].endswith("not_issued")), reverse=True)
    print("  top stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={int(v)}" for v, k in st[:6]))
