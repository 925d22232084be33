"""Print the key throughput / stall metrics of ncu reports (run where ncu is).

    python tools/ncu_keys.py gpurun_out/prof_*.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__inst_executed.sum")

for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        print(rep, "no data")
        continue
    hdr, units, vals = rows[0], rows[1], rows[2]
    print("==", rep, vals[hdr.index("Kernel Name")][:90] if "Kernel Name" in hdr else "")
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            print(f"  {h} = {v} {u}")
        elif "warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            try:
                if float(v) > 0.3:
                    print(f"  stall {h.split('stalled_')[1].split('_per')[0]} = {v}")
            except ValueError:
                pass
