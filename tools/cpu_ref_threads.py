"""Reference CPU HE Mul on the GPU box's host: 1 thread and all threads,
radix 2 (the reference default, tools/hemul.cpp:141) and radix 16 (the
fastest single-thread variant), for the single-GPU latency
comparison (the 134x gate is against the fastest single-thread time).

    python tools/cpu_ref_threads.py [--configs X M] [--out FILE]

Test / measurement infrastructure: runs oracle/_ref (the reference built from
its own sources), never the product path. One HE Mul per point, level warmed
outside the timing (bench.cpp:68-69).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["X", "M"])
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import bench
    from oracle_lib import Reference

    ref = Reference()
    nproc = os.cpu_count() or 1
    rows = []
    for name in args.configs:
        cfg = bench.CONFIGS[name]
        for threads in (1, nproc):
            for radix_log in (1, 4):
                t0 = time.time()
                ms, dig = ref.time_he_mul(*cfg, seed=1, reps=1, threads=threads,
                                          radix_log=radix_log)
                rows.append({"config": name, "threads": threads, "radix": 1 << radix_log,
                             "ms_per_he_mul": ms, "digest": f"{dig:016x}",
                             "wall_s": round(time.time() - t0, 1)})
                print(json.dumps(rows[-1]), flush=True)
    out = {"cpu_model": cpu_model(), "nproc": nproc, "results": rows}
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
