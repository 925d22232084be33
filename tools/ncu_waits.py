"""List the mbarrier wait sites of one ncu report (launch 0) with their
executions and retry counts — which role of a warp-specialised kernel waits
on which barrier (tools for kernel iteration).

    python tools/ncu_waits.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--print-source", "sass",
                      "--csv"], capture_output=True, text=True).stdout
src = list(csv.reader(io.StringIO(out)))
blocks = [i for i, row in enumerate(src) if row and row[0] == "Address"]
b = blocks[-1] if len(sys.argv) < 3 else blocks[int(sys.argv[2])]
h = src[b]
ei = h.index("Instructions Executed")
si = h.index("Warp Stall Sampling (All Samples)")
tot = 0
rows = [r for r in src[b + 1:] if len(r) > si]
for r in rows:
    try:
        tot += int(r[si] or 0)
    except ValueError:
        pass
for r in rows:
    t = r[1]
    if "SYNCS" in t or "UTCIMMA" in t or "UTMALDG" in t or "LDTM" in t or "NANOSLEEP" in t:
        n = int(r[ei] or 0)
        if n:
            print(f"{r[0][-5:]} {n:>11} {100 * int(r[si] or 0) / tot:5.1f}%  {t[:70]}")
