"""Quick look at an ncu report: per-launch headline metrics, stall reasons and
the SASS lines with the most stall samples (tools for kernel iteration).

    python tools/ncu_quick.py gpurun_out/prof.ncu-rep [--top 25]
"""
from __future__ import annotations

import argparse
import csv
import io
import subprocess

HEAD = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Memory Throughput", "L2 Hit Rate",
        "L1/TEX Hit Rate", "Registers Per Thread", "Achieved Active Warps Per SM"]


def run(args: list[str]) -> list[list[str]]:
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    r = run([a.report, "--page", "details"])
    h = r[0]
    idi, mi, vi, ui = h.index("ID"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    ki = h.index("Kernel Name")
    seen = {}
    for row in r[1:]:
        if row[mi] in HEAD:
            seen.setdefault((row[idi], row[ki][:60]), []).append(f"{row[mi]}={row[vi]}{row[ui]}")
    for k, v in seen.items():
        print(k[0], k[1])
        print("   " + "; ".join(v))
    raw = run([a.report, "--page", "raw"])
    hdr = raw[0]
    for row in raw[2:]:
        st = []
        for i, name in enumerate(hdr):
            if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
                try:
                    x = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                if x > 0:
                    st.append((x, name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        st.sort(reverse=True)
        tot = sum(x for x, _ in st) or 1
        print("stalls:", ", ".join(f"{n} {100 * x / tot:.0f}%" for x, n in st[:8]))
    src = run([a.report, "--page", "source", "--print-source", "sass"])
    blocks = [i for i, row in enumerate(src) if row and row[0] == "Address"]
    for bi, b0 in enumerate(blocks):
        hh = src[b0]
        si = hh.index("Warp Stall Sampling (All Samples)")
        ei = hh.index("Instructions Executed")
        end = blocks[bi + 1] - 1 if bi + 1 < len(blocks) else len(src)
        rows = []
        for row in src[b0 + 1:end]:
            try:
                rows.append((int(row[si]), row[0][-5:], row[ei], row[1]))
            except (ValueError, IndexError):
                pass
        tot = sum(x[0] for x in rows) or 1
        print(f"--- launch {bi}: top stall lines ({tot} samples)")
        for x in sorted(rows, reverse=True)[:a.top]:
            print(f"{100 * x[0] / tot:5.1f}% {x[1]} {x[2]:>10} {x[3][:100]}")


if __name__ == "__main__":
    main()
