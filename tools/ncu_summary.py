"""Summarise ncu reports into profiles/ (run here, on the reports gpurun brought back).

    python tools/ncu_summary.py gpurun_out/prof_*.ncu-rep --out profiles/r01_ncu_summary.md \
        --traffic profiles/traffic.json --config X

For each report (one kernel launch captured with --set full): duration, DRAM
bytes read+written (the `traffic` field of bench.py's roofline), pipe
utilisations (FMA-heavy = IMAD.WIDE, ALU, LSU), issue activity, occupancy,
shared-memory bank conflicts, registers.
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from pathlib import Path

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "fmaheavy_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_pct",
}

# ncu reports these in scaled units; normalise to bytes / milliseconds
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3,
        "ms": 1.0}


def read(rep: Path) -> dict:
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    res = {"kernel": vals[hdr.index("Kernel Name")]}
    for m, key in METRICS.items():
        # some sections prefix their metrics (e.g. "TPC.TriageCompute.")
        for i in [i for i, h in enumerate(hdr) if h == m or h.endswith("." + m)]:
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            res[key] = v * UNIT.get(units[i], 1.0)
            break
    return res


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("reports", nargs="+", type=Path)
    ap.add_argument("--out", type=Path, required=True)
    ap.add_argument("--traffic", type=Path)
    ap.add_argument("--config", default="X")
    ap.add_argument("--title", default="ncu --set full, one launch per kernel")
    args = ap.parse_args()
    lines = [f"# {args.title}", "",
             "| class | kernel | ms | DRAM read MB | DRAM write MB | tensor % | L2 % | FMA-heavy % | ALU % "
             "| LSU % | issue % | occupancy % | smem conflicts / wavefronts | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic = json.loads(args.traffic.read_text()) if args.traffic and args.traffic.exists() else {}
    for rep in args.reports:
        r = read(rep)
        name = r["kernel"].split("(")[0].split("::")[-1]
        key = rep.stem.split("prof_", 1)[-1]  # report named prof_<bench kernel class>.ncu-rep
        lines.append(
            f"| {key} | `{name}` | {r.get('duration', 0):.3f} | {r.get('dram_read', 0) / 1e6:.1f} | "
            f"{r.get('dram_write', 0) / 1e6:.1f} | {r.get('tensor_pct', 0):.1f} | "
            f"{r.get('l2_pct', 0):.1f} | {r.get('fmaheavy_pct', 0):.1f} | "
            f"{r.get('alu_pct', 0):.1f} | {r.get('lsu_pct', 0):.1f} | {r.get('issue_pct', 0):.1f} | "
            f"{r.get('occupancy_pct', 0):.1f} | {r.get('smem_conflicts', 0):.3g} / "
            f"{r.get('smem_wavefronts', 0):.3g} | {int(r.get('regs', 0))} | "
            f"{int(r.get('grid', 0))} x {int(r.get('block', 0))} |")
        traffic.setdefault(args.config, {})[key] = r.get("dram_read", 0) + r.get("dram_write", 0)
    args.out.write_text("\n".join(lines) + "\n")
    if args.traffic:
        args.traffic.write_text(json.dumps(traffic, indent=1, sort_keys=True) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
