"""BASELINE config C2: standalone batched NTT / iNTT sweep on one B200.

    python tools/ntt_sweep.py [--out profiles/r01_ntt_sweep.json] [--cpu]

For logN in 12..17 and prime counts np in {4, 5, 7, 42, 63, 84, 125}
(SURVEY.md §8(d) C2): forward and inverse negacyclic NTT over `batch x np`
prime-major rows of random residues, through the stage entry point
hemul_gpu_ntt (= ntt_forward / ntt_inverse, ntt.cpp:153-197), device-resident
inputs, CUDA events, median of 10. Reports ms per call, butterflies/s and
the IMAD roofline fraction (9 IMAD-equivalents per Shoup butterfly). The
reference's single-thread CPU NTT on the same shapes is in SURVEY.md
Appendix B (5-10 ns per butterfly).
"""
from __future__ import annotations

import argparse
import json
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
    ap.add_argument("--batch", type=int, default=8)
    args = ap.parse_args()
    import torch

    from paper_2003_04510_b200.hemul import Context, make_params

    results = []
    peak = None
    for log_n in range(12, 18):
        # depth 80 at this ring degree: region 2 holds >= 125 primes
        ctx = Context(make_params(30, 80, log_n))
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
        ctx.set_stream(stream.cuda_stream)
        if peak is None:
            peak = ctx.imad_peak()
        q = ctx.params.log_q_max
        primes = ctx.level_primes(q, 2)
        n = 1 << log_n
        for npr in NPS:
            rows = npr * args.batch
            p = torch.tensor(primes[np.arange(rows) % len(primes)].astype(np.int64),
                             device="cuda").view(-1, 1)
            data = (torch.randint(0, 2**62, (rows, n), device="cuda", dtype=torch.int64) % p)
            data = data.view(torch.uint64).contiguous()
            rec = {"log_n": log_n, "np": npr, "batch": args.batch, "rows": rows}
            for inverse in (False, True):
                for _ in range(3):
                    ctx.ntt(data, q, 2, inverse=inverse)
                times = []
                for _ in range(10):
                    a = torch.cuda.Event(enable_timing=True)
                    b = torch.cuda.Event(enable_timing=True)
                    a.record(stream)
                    ctx.ntt(data, q, 2, inverse=inverse)
                    b.record(stream)
                    torch.cuda.synchronize()
                    times.append(a.elapsed_time(b))
                ms = statistics.median(times)
                bfly = rows * (n // 2) * log_n
                key = "inv" if inverse else "fwd"
                rec[f"{key}_ms"] = ms
                rec[f"{key}_gbfly_s"] = bfly / (ms * 1e-3) / 1e9
                rec[f"{key}_imad_frac"] = 9 * bfly / (ms * 1e-3) / peak
            results.append(rec)
            print(json.dumps(rec), flush=True)
        ctx.close()
    args.out.write_text(json.dumps({"imad_peak_ops": peak, "results": results}, indent=1) + "\n")


if __name__ == "__main__":
    main()
