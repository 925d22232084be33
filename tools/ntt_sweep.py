"""BASELINE config C2: standalone batched NTT / iNTT sweep on one B200.

    python tools/ntt_sweep.py [--out profiles/r02_ntt_sweep.json] [--no-cpu]

For logN in 12..17 and prime counts np in {4, 5, 7, 42, 63, 84, 125}
(bench_ntt.cpp:10-27): forward and inverse negacyclic NTT
over `batch x np` prime-major rows through hemul_gpu_ntt32, i.e. the 30-bit
basis kernels of the he_mul path (ntt_col.cu pass A + the block pass B; the
evk forms take exactly this path, he_mul fuses pass B into ntt_blk.cu).
Batches 1 and 8. Device-resident u32 rows, CUDA events, median of 10.

Per point:
  ms, Gbutterflies/s, HBM GB/s and fraction of MEASURED_PEAKS.json (each of
  the two memory passes reads and writes every row once: 16 bytes per
  residue), a parity check of every row of the batch-1 run against the C
  restatement (oracle/hemul_oracle.c orc_ntt_forward / orc_ntt_inverse with
  the same primes and min-root rule; lazy GPU outputs compared mod p), and
  the reference's own CPU ntt_forward / ntt_inverse (oracle/_ref, w64
  primes, radix 16, bench_ntt.cpp protocol) at 1 and nproc threads on this
  host, same (logN, np).

Test / measurement infrastructure: the oracle and oracle/_ref are only the
checker and the CPU baseline here, never the measured GPU path.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "tests")]

NPS = (4, 5, 7, 42, 63, 84, 125)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", type=Path, default=ROOT / "profiles" / "ntt_sweep.json")
    ap.add_argument("--log-n", type=int, nargs="+", default=list(range(12, 18)))
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import torch

    import bench
    import modmath as mm
    from oracle_lib import REFERENCE_SO, Reference, Restated
    from paper_2003_04510_b200.hemul import Context, make_params

    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    hbm_peak = peaks.get("hbm_gbs")
    restated = Restated()
    ref = Reference() if (REFERENCE_SO.exists() and not args.no_cpu) else None
    nproc = os.cpu_count() or 1
    results = []
    for log_n in args.log_n:
        # depth 80: region 2 of the fresh level holds >= 125 30-bit primes
        ctx = Context(make_params(30, 80, log_n))
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        ctx.set_stream(stream.cuda_stream)
        ctx.set_basis(32)
        q = ctx.params.log_q_max
        primes = ctx.level_primes(q, -2)
        assert len(primes) >= max(NPS), len(primes)
        n = 1 << log_n
        for npr in NPS:
            rec = {"log_n": log_n, "np": npr}
            ps = primes[:npr]
            pt = torch.tensor(ps.astype(np.int64), device="cuda").view(-1, 1)
            for batch in (1, 8):
                rows = npr * batch  # row r mod ps[r % npr] (hemul_gpu_ntt32 np = npr)
                g = torch.Generator(device="cuda")
                g.manual_seed(3 + log_n * 1000 + npr)
                vals = torch.randint(0, 2**31, (rows, n), generator=g, device="cuda",
                                     dtype=torch.int64) % pt.repeat(batch, 1)
                data = vals.to(torch.int32).contiguous()
                x0 = vals.cpu().numpy().astype(np.uint64)
                for inverse in (False, True):
                    work = data.clone()
                    ctx.ntt32(work, q, 2, inverse=inverse, nprimes=npr)  # warm + parity
                    if batch == 1:
                        got = work.cpu().numpy().view(np.uint32).astype(np.uint64)
                        roots = [mm.root_2n(int(p), n) for p in ps]
                        want = restated.ntt(x0, ps, roots, log_n, inverse=inverse)
                        P = ps.astype(np.uint64)[:, None]
                        ok = bool(np.array_equal(got % P, want % P))
                        rec[f"{'inv' if inverse else 'fwd'}_parity"] = ok
                        assert ok, (log_n, npr, inverse)
                    ts = []
                    for _ in range(args.reps):
                        e0 = torch.cuda.Event(enable_timing=True)
                        e1 = torch.cuda.Event(enable_timing=True)
                        e0.record(stream)
                        ctx.ntt32(work, q, 2, inverse=inverse, nprimes=npr)
                        e1.record(stream)
                        torch.cuda.synchronize()
                        ts.append(e0.elapsed_time(e1))
                    ms = statistics.median(ts)
                    byts = 2 * 2 * rows * n * 4  # two memory passes, read + write
                    bfly = rows * (n // 2) * log_n
                    rec[f"{'inv' if inverse else 'fwd'}_b{batch}"] = {
                        "ms": ms, "rows": rows, "gbutterflies_s": bfly / ms / 1e6,
                        "hbm_gbs": byts / ms / 1e6,
                        "hbm_frac": (byts / ms / 1e6 / hbm_peak) if hbm_peak else None}
            if ref is not None:
                for inverse in (False, True):
                    for threads in (1, nproc):
                        t = ref.time_ntt(log_n, npr, threads=threads,
                                         radix_log=bench.FASTEST_RADIX_LOG, reps=3,
                                         inverse=inverse)
                        rec[f"cpu_{'inv' if inverse else 'fwd'}_t{threads}_ms"] = statistics.median(t)
            results.append(rec)
            print(json.dumps(rec), flush=True)
        ctx.close()
    out = {"config": "C2", "basis": "30-bit (he_mul path kernels)", "hbm_peak_gbs": hbm_peak,
           "cpu": {**bench.cpu_info(), "radix": 1 << bench.FASTEST_RADIX_LOG,
                   "primes": "w64 generate_primes (reference)"},
           "results": results}
    args.out.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
