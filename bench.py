"""HE Mul (+ relinearize + rescale) benchmark — BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config X|M|S]
                    [--batch B] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (N > 1)

One step = one batched call of the reference-facing entry point
(hemul_gpu_he_mul, include/hemul_gpu.h == Scheme::he_mul, heaan.cpp:339-410)
on B independent ciphertext pairs per GPU at the fresh modulus of the
config (default X: N=2^17, logQ=2400 — the paper-scale point the metric is
quoted on). Independent HE Muls shard by ciphertext across GPUs (weak
scaling, replicated evk, no collective inside the timed region; NCCL only
takes the max of the per-rank times and gathers result digests afterwards).

Printed JSON (rank 0, one line):
  value     whole-job HE Mul/s with inputs resident in HBM (device event time,
            max over ranks)
  latency_us  single HE Mul (batch 1) device latency on rank 0
  e2e       the same metric through the C-ABI with pinned HOST buffers: every
            step copies its inputs H2D and its outputs D2H inside the timed
            region
  roofline  dominant kernel class of the timed region against its bound:
            NTT passes = HBM bytes vs MEASURED_PEAKS.json; base-conversion
            GEMMs = algorithmic u8 MACs vs the int8 tensor-core peak measured
            on this device in this run (tcgen05 probe; or IMAD.WIDE products
            vs the IMAD probe with --engine imad). `kernels` lists every class.
  cpu_baseline  the reference CPU he_mul (oracle/_ref, compiled from the
            reference sources) in its fastest variant (NTT radix 16) on this
            host: 1 HE Mul on all cores (value) + 1 on one thread (latency
            comparison), CPU model and clock; --cpu-full adds the full
            protocol (3 reps x radix 2/16 x 1/all threads)
--impl reference times that same reference CPU implementation (fastest
variant, all host threads) as the whole arm, on the same config and metric.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = ("HE Mul latency (µs) at N=2^17; batched HE Mul/s at 1/2/4/8 B200 vs CPU ref")
CONFIGS = {  # make_params(log_p, depth, w64, log_n_override)
    "X": (30, 80, 0),   # N=2^17, logQ=2400 (paper scale; BASELINE configs[3,4])
    "M": (30, 40, 0),   # N=2^16, logQ=1200 (paper Table 7 point)
    "S": (30, 4, 13),   # N=2^13, logQ=120
}
DEFAULT_BATCH = {"X": 8, "M": 16, "S": 64}


def limbs(bits: int) -> int:
    return (bits + 63) // 64


# --------------------------------------------------------------------------
# algorithmic work per kernel class
# --------------------------------------------------------------------------
GEMM_CLASSES = ("crt", "icrt", "finish")     # bound: int8 tensor cores (or IMAD.WIDE.U32)
NTT_CLASSES = ("ntt_a", "ntt_b", "intt_b", "intt_a", "mid_r1", "mid_r2", "tensor", "evk")


def split_point(log_q: int) -> int:
    """level_tables.hpp split_point: ceil(log_q/2) rounded up to a byte."""
    h = (log_q + 1) // 2
    h8 = (h + 7) // 8 * 8
    return h8 if h8 < log_q else h


def kernel_model(p, word: int, np1: int, np2: int, B: int, log_q: int,
                 tensor: bool = False) -> dict[str, dict]:
    """Per kernel class and step: `products` = the algorithmic inner-product
    terms of the integer GEMMs on the IMAD pipe (one IMAD.WIDE.U32 each:
    25-bit chunk x 30-bit operand), or with `tensor` (30-bit basis, int8
    tensor cores) `macs` = the algorithmic u8 x u8 multiply-accumulates
    (byte planes x bytes; padding not counted); `bytes` = the
    HBM bytes the kernel must move (each operand read once, each result
    written once); `butterflies` = NTT butterflies. word 32: the 30-bit
    basis with split region 1 (np1 primes per half product); word 64: the
    reference's w64 basis."""
    n, ln = p.n, p.log_n
    s1 = ln if ln <= 11 else (ln + 1) // 2
    s2 = ln - s1
    L = limbs(log_q)
    kq = math.ceil(log_q / 25)
    fin_cols = math.ceil((min(p.log_q_max, 125) + log_q) / 25)
    rb = n * word // 8                       # bytes of one RNS row
    if word == 32:
        h = (log_q + 1) // 2
        in1, out1, R = 8, 6, 1
        crt_products = n * B * (8 * math.ceil(h / 25) * np1 + kq * np2)
    else:
        in1, out1, R = 4, 3, 2
        crt_products = n * B * (4 * np1 + np2) * 2 * kq
    k1 = (R * np1 + 1) * (2 if word == 32 else 1)
    k2 = R * np2 + 1
    fwd_rows = in1 * B * np1 + B * np2
    inv_rows = out1 * B * np1 + 2 * B * np2
    bf = n // 2
    if tensor and word == 32:
        h = split_point(log_q)
        T2 = log_q + p.log_q_max
        base8 = max(0, p.log_q_max - 125) // 8 * 8
        crt_macs = n * B * (8 * math.ceil(h / 8) * 4 * np1 + math.ceil(log_q / 8) * 4 * np2)
        icrt_macs = n * B * (4 * 2 * np1 + 7) * math.ceil(log_q / 8)
        fin_macs = n * 2 * B * (4 * (np2 + 2 * np1) + 7) * math.ceil((T2 - base8) / 8)
    m = {
        "crt": {"products": crt_products,
                "bytes": 5 * B * n * L * 8 + fwd_rows * rb},
        "icrt": {"products": n * B * k1 * kq,
                 "bytes": (2 if word == 32 else 1) * B * np1 * rb + B * n * L * 8},
        "finish": {"products": n * 2 * B * (k2 + k1) * fin_cols,
                   "bytes": 2 * B * np2 * rb + (out1 - 2) * B * np1 * rb
                            + 2 * B * n * limbs(log_q - p.log_p) * 8},
        "ntt_a": {"butterflies": fwd_rows * bf * s1, "bytes": 2 * fwd_rows * rb},
        "intt_a": {"butterflies": inv_rows * bf * s1, "bytes": 2 * inv_rows * rb},
        "ntt_b": {"butterflies": fwd_rows * bf * s2, "bytes": 2 * fwd_rows * rb},
        "intt_b": {"butterflies": inv_rows * bf * s2, "bytes": 2 * inv_rows * rb},
        "mid_r1": {"butterflies": (in1 + out1) * B * np1 * bf * s2,
                   "bytes": (in1 + out1) * B * np1 * rb},
        "mid_r2": {"butterflies": 3 * B * np2 * bf * s2,
                   "bytes": 3 * B * np2 * rb + 2 * np2 * rb},
        "tensor": {"bytes": (in1 + out1) * B * np1 * rb},
        "evk": {"bytes": 3 * B * np2 * rb + 2 * np2 * rb},
    }
    if tensor and word == 32:
        for k, v in (("crt", crt_macs), ("icrt", icrt_macs), ("finish", fin_macs)):
            del m[k]["products"]
            m[k]["macs"] = v
    return m


# --------------------------------------------------------------------------
# clocks sampler (B200_PROFILING.md)
# --------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled through NVML every ~2 ms while the
    timed region runs (the timed region can be ~100 ms, too short for
    `nvidia-smi -lms`); falls back to nvidia-smi when NVML is unavailable."""
    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}
    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int, period_s: float = 0.002):
        self.device = device
        self.period = period_s
        self.sm: list[float] = []
        self.max_mhz = None
        self.reasons: set[str] = set()
        self.proc = None
        self.lines: list[str] = []
        self._stop = threading.Event()
        self._nvml = None

    def _handle(self):
        import pynvml

        pynvml.nvmlInit()
        try:
            import torch

            uuid = str(torch.cuda.get_device_properties(self.device).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID(
                uuid if uuid.startswith("GPU-") else "GPU-" + uuid)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _poll(self):
        nv, h = self._nvml
        masks = {k: getattr(nv, v) for k, v in self.REASONS.items()}
        while True:
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for k, m in masks.items():
                    if r & m:
                        self.reasons.add(k)
            except Exception:
                pass
            if self._stop.wait(self.period):
                return

    def __enter__(self):
        try:
            self._nvml = self._handle()
            nv, h = self._nvml
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self._nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self._nvml is not None:
            self._stop.set()
            self.thread.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = list(self.sm), self.max_mhz, set(self.reasons)
        names = list(self.REASONS)
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


# --------------------------------------------------------------------------
# reference CPU arm / baseline
# --------------------------------------------------------------------------
# The reference's fastest NTT variant on this host (SURVEY.md §8(d):
# radix 2^4 beats the default radix 2 by 11-27 %, profiles/r01_cpu_ref_threads.json);
# both the cpu_baseline leg and the reference arm use it.
FASTEST_RADIX_LOG = 4


def cpu_info() -> dict:
    """CPU model, logical cores and the current clock (median of /proc/cpuinfo)."""
    model, mhz = platform.processor(), []
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
            elif line.startswith("cpu MHz"):
                mhz.append(float(line.split(":", 1)[1]))
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count() or 1,
            "cpu_mhz": statistics.median(mhz) if mhz else None}


def reference_cpu(cfg, reps: int, threads: int, seed: int = 1,
                  radix_log: int = FASTEST_RADIX_LOG):
    sys.path.insert(0, str(ROOT / "tests"))
    from oracle_lib import REFERENCE_SO, Reference

    if not REFERENCE_SO.exists():
        return None, "oracle/_ref/libhemul_ref.so missing (build it where /root/reference exists)"
    ref = Reference()
    t0 = time.time()
    ms, dig = ref.time_he_mul(*cfg, seed=seed, reps=reps, threads=threads, radix_log=radix_log)
    return {"ms": ms, "digest": f"{dig:016x}", "wall_s": time.time() - t0}, None


def reference_cpu_full(cfg, reps: int = 3) -> dict:
    """SURVEY.md §8(d) CPU protocol: `reps` HE Muls at radix 2 (the reference
    default, tools/hemul.cpp:141) and radix 16, on 1 thread and on all threads."""
    nproc = os.cpu_count() or 1
    rows = []
    for threads in (1, nproc):
        for radix_log in (1, 4):
            res, why = reference_cpu(cfg, reps=reps, threads=threads, radix_log=radix_log)
            if res is None:
                return {"unavailable": why}
            rows.append({"threads": threads, "radix": 1 << radix_log, "ms": res["ms"],
                         "ms_median": statistics.median(res["ms"]), "digest": res["digest"]})
            print(json.dumps(rows[-1]), file=sys.stderr, flush=True)
    single = min((r for r in rows if r["threads"] == 1), key=lambda r: r["ms_median"])
    return {**cpu_info(), "reps": reps, "results": rows,
            "fastest_single_thread_ms": single["ms_median"],
            "fastest_single_thread_radix": single["radix"]}


STAGE_MAP = {
    "crt": "crt_forward of region 1 (8 half-inputs) and region 2 (ModUp of d2)",
    "ntt": "forward pass A + the fused middle passes (forward tails, the pointwise "
           "tensor / evk products the reference books under iCRT, inverse heads)",
    "intt": "inverse pass A (emits t_j = x (P/p_j)^-1)",
    "icrt": "iCRT of d2 + the fused finisher (ModDown, d0/d1 add, rescale: the "
            "reference's Extra work)",
    "extra": "0: poly_add/sub/shift are fused into the finisher (icrt)",
}


def poly_source(n: int, seed: int, device: str = "cuda"):
    """rand_poly(batch, bits): uniform BigPolys (batch, n, limbs) mod 2^bits
    from one seeded device generator."""
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)

    def rand_poly(batch, bits):
        t = torch.randint(-(2**63), 2**63 - 1, (batch, n, limbs(bits)), generator=g,
                          device=device, dtype=torch.int64)
        if bits % 64:
            t[..., -1] &= (1 << (bits % 64)) - 1
        return t.view(torch.uint64)

    return rand_poly


def make_inputs(n: int, q: int, B: int, seed: int, device: str = "cuda"):
    """The bench's synthetic inputs (rank r uses seed 1000 + r): B ciphertext
    pairs mod 2^q and an evk mod 2^(2q), uniform limbs, top limb masked."""
    rand_poly = poly_source(n, seed, device)
    c1 = (rand_poly(B, q), rand_poly(B, q))
    c2 = (rand_poly(B, q), rand_poly(B, q))
    evk = (rand_poly(1, 2 * q)[0].contiguous(), rand_poly(1, 2 * q)[0].contiguous())
    return c1, c2, evk


def run_reference_arm(args, cfg, rank: int) -> None:
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    # one step = one full HE Mul (fastest variant, all host threads); warm-up
    # steps run untimed
    res, why = reference_cpu(cfg, reps=args.warmup + args.steps, threads=threads)
    if res is None:
        print(json.dumps({"impl": "reference", "unavailable": why}))
        return
    timed = res["ms"][args.warmup:]
    ms = statistics.mean(timed)
    value = 1000.0 / ms
    from paper_2003_04510_b200.hemul import make_params

    p = make_params(*cfg)
    sample = (f"{args.steps} timed + {args.warmup} warm-up reference Scheme::he_mul calls "
              f"(N=2^{p.log_n}, logQ={p.log_q_max}, NTT radix {1 << FASTEST_RADIX_LOG}, the "
              f"fastest variant), random inputs, level warmed outside timing")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "HE Mul/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "latency_us": ms * 1000.0, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.config}: HE Mul N=2^{p.log_n} logQ={p.log_q_max}",
                   "batch_per_gpu": 1, "threads": threads,
                   "radix": 1 << FASTEST_RADIX_LOG},
        "cpu_baseline": {"value": value, "unit": "HE Mul/s", "cores": threads,
                         "kind": "reference", "sample": sample, **cpu_info()},
        "e2e": {"value": value, "unit": "HE Mul/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "digest": res["digest"],
    }))


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------
def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="X", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0, help="HE Muls per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-full", action="store_true",
                    help="also run the full CPU protocol (3 reps, radix 2/16, 1/all threads; "
                         "several minutes at X) into cpu_baseline.full")
    ap.add_argument("--latency-reps", type=int, default=5)
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: the same code path without "
                         "NCCL, e.g. for two ranks sharing one GPU in tests)")
    ap.add_argument("--one-device", action="store_true",
                    help="every rank on cuda:0 (exercises the multi-rank path on one GPU)")
    ap.add_argument("--chain", type=int, default=8,
                    help="device-resident chain length for the `chain` key (0 = skip)")
    ap.add_argument("--levels", default="0.5,0.25",
                    help="fractions of log Q at which to time device-resident batches for the "
                         "`lower_levels` key (empty = skip)")
    ap.add_argument("--basis", type=int, default=32, choices=[32, 64],
                    help="RNS basis of he_mul (HEMUL_OPT_BASIS); results are identical")
    ap.add_argument("--engine", default="tc", choices=["tc", "imad"],
                    help="30-bit basis base conversions on the int8 tensor cores (tc) or the "
                         "IMAD.WIDE pipe (HEMUL_OPT_TENSOR_CORES); results are identical")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    B = args.batch or DEFAULT_BATCH[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference_arm(args, cfg, rank)
        return

    import torch
    import torch.distributed as dist

    from paper_2003_04510_b200.dist import gather_to_rank0, max_over_ranks
    from paper_2003_04510_b200.hemul import Context, ciphertext_digest, make_params

    if args.one_device:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    p = make_params(*cfg)
    ctx = Context(p, device=local)
    # a dedicated (non-legacy) stream shared by torch and the library, so the
    # CUDA events below bracket the library's kernels
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_basis(args.basis)
    ctx.set_tensor_cores(args.engine == "tc")
    if os.environ.get("HEMUL_BENCH_TRANSPOSED"):
        ctx.set_transposed(os.environ["HEMUL_BENCH_TRANSPOSED"] == "1")
    q = p.log_q_max
    L, Lo, Le = limbs(q), limbs(q - p.log_p), limbs(2 * q)
    n = p.n

    # synthetic random ciphertexts and keys (SURVEY §8(d) throughput inputs),
    # generated on the device, resident before timing; per-rank seeds
    c1, c2, evk = make_inputs(n, q, B, seed=1000 + rank)
    out = (torch.empty((B, n, Lo), dtype=torch.uint64, device="cuda"),
           torch.empty((B, n, Lo), dtype=torch.uint64, device="cuda"))
    t0 = time.time()
    ctx.warm_level(q, evk, evk_id=1)
    level_s = time.time() - t0
    word, np1, np2 = ctx.mul_basis(q)   # the RNS basis he_mul runs in

    def step(b=B, o=out):
        ctx.he_mul((c1[0][:b], c1[1][:b]), (c2[0][:b], c2[1][:b]), q, evk=evk, evk_id=1,
                   out=(o[0][:b], o[1][:b]))

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- warm-up ---------------------------------------------------------
    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()

    # ---- headline timed region: device-resident inputs --------------------
    ctx.enable_stage_timing(True)
    ctx.reset_stats()
    launches0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    launches = ctx.launch_count() - launches0
    kstats = ctx.kernel_stats()
    ctx.enable_stage_timing(False)
    elapsed_ms = max_over_ranks(elapsed_ms, device="cuda")
    value = world * B * args.steps / (elapsed_ms / 1000.0)
    ms_per_step = elapsed_ms / args.steps

    # ---- single HE Mul latency (batch 1) ----------------------------------
    lat = []
    for _ in range(args.latency_reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step(1)
        b.record(stream)
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b) * 1000.0)
    latency_us = statistics.median(lat)

    # ---- stage breakdown of one HE Mul (reference buckets) ----------------
    ctx.enable_stage_timing(True)
    step()
    stage_ms = ctx.stage_ms()
    ctx.enable_stage_timing(False)

    # ---- e2e through the C-ABI with pinned host buffers --------------------
    hc1 = tuple(x.cpu().pin_memory() for x in c1)
    hc2 = tuple(x.cpu().pin_memory() for x in c2)
    ho = tuple(torch.empty((B, n, Lo), dtype=torch.uint64).pin_memory() for _ in range(2))
    nph = lambda t: t.numpy()  # noqa: E731 — pinned tensors viewed as host arrays

    def e2e_step():
        ctx.he_mul((nph(hc1[0]), nph(hc1[1])), (nph(hc2[0]), nph(hc2[1])), q, evk=evk,
                   evk_id=1, out=(nph(ho[0]), nph(ho[1])))

    e2e_step()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_ms = max_over_ranks(e2e_ms, device="cuda")
    e2e_value = world * B * e2e_steps / (e2e_ms / 1000.0)
    if not torch.equal(ho[0], out[0].cpu()) and not os.environ.get("HEMUL_BENCH_ABLATION"):
        raise RuntimeError("e2e output differs from the device-resident output")

    # ---- device-resident chain: B accumulators times K
    # fresh ciphertexts down K levels (mod_down on the device), one upload of
    # every operand and one download of the result inside the timed region;
    # every level's tables and evk forms warmed by an untimed first pass
    K = args.chain
    chain = None
    if K > 0:
        ctx.set_level_cache(K + 1)
        rand_poly = poly_source(n, seed=2000 + rank)
        hf = [tuple(rand_poly(B, q).cpu().pin_memory() for _ in range(2)) for _ in range(K)]
        ha = (nph(hc1[0]), nph(hc1[1]))
        hres = tuple(torch.empty((B, n, limbs(q - K * p.log_p)), dtype=torch.uint64).pin_memory()
                     for _ in range(2))

        def run_chain():
            # pinned sources, queued on the copy stream: operand k+1 crosses
            # PCIe while HE Mul k runs
            acc = ctx.upload(ha, q, asynchronous=True)
            fresh = [ctx.upload((nph(f[0]), nph(f[1])), q, asynchronous=True) for f in hf]
            for f in fresh:
                f = ctx.mod_down_dev(f, acc.log_q) if f.log_q > acc.log_q else f
                acc = ctx.he_mul_dev(acc, f, evk=evk, evk_id=1)
            acc.download(out=(nph(hres[0]), nph(hres[1])))  # into pinned host buffers
            return acc.log_q

        run_chain()
        torch.cuda.synchronize()
        barrier()
        c0, c1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        final_q = run_chain()
        c1e.record(stream)
        torch.cuda.synchronize()
        chain_ms = max_over_ranks(c0.elapsed_time(c1e), device="cuda")
        chain = {"value": world * B * K / (chain_ms / 1000.0), "unit": "HE Mul/s",
                 "chain_len": K, "batch_per_gpu": B, "ms": chain_ms,
                 "levels": f"{q} -> {final_q}",
                 "h2d_bytes": (K + 1) * 2 * B * n * L * 8,
                 "d2h_bytes": 2 * B * n * limbs(final_q) * 8,
                 "note": "one H2D of every operand and one D2H of the result per chain "
                         "(hemul_gpu_ct_* handles); level LRU sized to the chain"}

    # ---- throughput below the fresh modulus: device-resident batches at a few
    # lower levels (region 2 of the 30-bit basis shrinks with the level: the
    # key is taken mod 2^(log_q + log_Q)); same batch, same key
    lower = []
    if args.levels:
        ctx.set_level_cache(2)
        for frac in (float(x) for x in args.levels.split(",")):
            lq = max(2 * p.log_p, int(q * frac) // p.log_p * p.log_p)
            lc1, lc2, _ = make_inputs(n, lq, B, seed=3000 + rank)
            lo = tuple(torch.empty((B, n, limbs(lq - p.log_p)), dtype=torch.uint64,
                                   device="cuda") for _ in range(2))
            ctx.warm_level(lq, evk, evk_id=1)

            def lstep():
                ctx.he_mul(lc1, lc2, lq, evk=evk, evk_id=1, out=lo)

            lstep()
            torch.cuda.synchronize()
            barrier()
            l0, l1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            l0.record(stream)
            lsteps = max(1, min(args.steps, 5))
            for _ in range(lsteps):
                lstep()
            l1.record(stream)
            torch.cuda.synchronize()
            lms = max_over_ranks(l0.elapsed_time(l1), device="cuda") / lsteps
            _, lnp1, lnp2 = ctx.mul_basis(lq)
            lower.append({"log_q": lq, "value": world * B / (lms / 1000.0), "unit": "HE Mul/s",
                          "ms_per_step": lms, "np1": lnp1, "np2": lnp2})

    # ---- result digests gathered to rank 0 (after timing) ------------------
    o0 = out[0][0].cpu().numpy(), out[1][0].cpu().numpy()
    dig = ciphertext_digest(q - p.log_p, o0[0], o0[1])
    digests = gather_to_rank0(dig) or []

    # ---- roofline: GEMM kernels vs the int8 tensor-core / IMAD.WIDE probes
    # measured on this device in this run, NTT kernels vs HBM
    imad_peak = ctx.imad_peak()
    tc_peak = ctx.tc_peak()
    tensor = args.engine == "tc" and word == 32
    peaks = {}
    pfile = ROOT / "MEASURED_PEAKS.json"
    if pfile.exists():
        peaks = json.loads(pfile.read_text())
    hbm_peak = peaks.get("hbm_gbs")
    model = kernel_model(p, word, np1, np2, B, q, tensor=tensor)
    per_class = {}
    for k, (ms, cnt) in kstats.items():
        if k not in model or ms <= 0:
            continue
        sec = ms / args.steps * 1e-3
        mk = model[k]
        e = {"ms_per_step": ms / args.steps, "launches_per_step": cnt / args.steps,
             "hbm_gbs": mk["bytes"] / sec / 1e9}
        if hbm_peak:
            e["hbm_frac"] = e["hbm_gbs"] / hbm_peak
        if "products" in mk:
            e["tiops"] = mk["products"] / sec / 1e12
            e["imad_frac"] = e["tiops"] / (imad_peak / 1e12)
        if "macs" in mk:
            e["tensor_tops"] = 2 * mk["macs"] / sec / 1e12
            e["tensor_frac"] = e["tensor_tops"] / (tc_peak / 1e12)
        if "butterflies" in mk:
            e["gbutterflies_s"] = mk["butterflies"] / sec / 1e9
        per_class[k] = e
    dom = max(per_class, key=lambda k: per_class[k]["ms_per_step"])
    traffic = None
    tfile = ROOT / "profiles" / "traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dom)
    if "tensor_tops" in per_class[dom]:
        roof = {"bound": "tensor", "kernel": dom, "achieved": per_class[dom]["tensor_tops"],
                "peak": tc_peak / 1e12, "unit": "TOP/s (int8, dense)",
                "frac": per_class[dom]["tensor_frac"], "traffic": traffic,
                "peak_source": "tcgen05.mma kind::i8 probe on this device, this run"}
    elif "tiops" in per_class[dom]:
        roof = {"bound": "imad", "kernel": dom, "achieved": per_class[dom]["tiops"],
                "peak": imad_peak / 1e12, "unit": "TIOP/s (IMAD.WIDE.U32 products)",
                "frac": per_class[dom]["imad_frac"], "traffic": traffic,
                "peak_source": "IMAD.WIDE.U32 probe on this device, this run"}
    else:
        roof = {"bound": "hbm", "kernel": dom, "achieved": per_class[dom]["hbm_gbs"],
                "peak": hbm_peak, "unit": "GB/s", "frac": per_class[dom].get("hbm_frac"),
                "traffic": traffic, "peak_source": "MEASURED_PEAKS.json hbm_gbs"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            # bounded sample (~25 s of CPU work at X): one HE Mul of the
            # reference's fastest variant on all host threads (the value) and
            # one on a single thread (the latency comparison)
            threads = os.cpu_count() or 1
            res, why = reference_cpu(cfg, reps=1, threads=threads)
            one, _ = reference_cpu(cfg, reps=1, threads=1) if res is not None else (None, None)
            if res is not None:
                v = 1000.0 / res["ms"][0]
                cpu = {"value": v, "unit": "HE Mul/s", "cores": threads, "kind": "reference",
                       "sample": f"1 reference Scheme::he_mul (N=2^{p.log_n}, logQ={q}, NTT radix "
                                 f"{1 << FASTEST_RADIX_LOG}) on {threads} threads and 1 on one "
                                 f"thread, random inputs, level warmed outside timing",
                       "latency_ms": res["ms"][0],
                       "single_thread_latency_ms": one["ms"][0] if one else None,
                       "radix": 1 << FASTEST_RADIX_LOG, **cpu_info()}
                if one:
                    cpu["gpu_latency_speedup_vs_single_thread"] = one["ms"][0] * 1000.0 / latency_us
                if args.cpu_full:
                    cpu["full"] = reference_cpu_full(cfg)
            else:
                cpu = {"value": None, "unavailable": why}
        line = {
            "metric": METRIC, "value": value, "unit": "HE Mul/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "latency_us": latency_us, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u32" if word == 32 else "u64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: batched HE Mul+relin+rescale, "
                                   f"N=2^{p.log_n}, logQ={q}, basis {word}-bit: np1={np1}"
                                   f"{' per half product' if word == 32 else ''}, np2={np2}",
                       "batch_per_gpu": B, "global_batch": B * world,
                       "parallelism": f"ciphertext-sharded x{world}, evk replicated",
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "seeds": f"rank r: inputs seed 1000 + r (bench.make_inputs)",
                       "l2": f"inputs {4 * B * n * L * 8 / 2**20:.0f} MiB per step > 126 MiB L2"},
            "gpu_launches": launches,
            "e2e": {"value": e2e_value, "unit": "HE Mul/s",
                    "h2d_bytes_per_step": 4 * B * n * L * 8,
                    "d2h_bytes_per_step": 2 * B * n * Lo * 8},
            "chain": chain,
            "lower_levels": lower,
            "roofline": roof,
            "kernels": per_class,
            "engine": "int8 tensor cores (tcgen05)" if tensor else "IMAD.WIDE integer pipe",
            "peaks": {"tensor_int8_tops": tc_peak / 1e12, "imad_wide_tops": imad_peak / 1e12,
                      "hbm_gbs": hbm_peak},
            "stage_ms_one_call": stage_ms,
            # our buckets vs the reference's StageTimers (counters.hpp, rns.cpp:364,
            # bench.cpp:81-84: pointwise booked under iCRT, add/sub/shift under Extra)
            "stage_map": STAGE_MAP,
            "level_setup_s": level_s,
            "clocks": clocks.summary(),
            "cpu_baseline": cpu,
            "digests": [f"{d:016x}" for d in digests],
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    ctx.close()


if __name__ == "__main__":
    main()
