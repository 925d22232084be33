"""Where the time of bench.py's device-resident chain goes (X, B=8, K=8):
upload only, compute only (operands already resident), and the full chain
with synchronous and asynchronous uploads. Prints one JSON line."""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2003_04510_b200.hemul import Context, make_params  # noqa: E402


def main() -> None:
    B, K = 8, 8
    p = make_params(30, 80, 0)
    q, n = p.log_q_max, p.n
    L = (q + 63) // 64
    ctx = Context(p)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    ctx.set_level_cache(K + 1)
    g = torch.Generator().manual_seed(1)

    def rnd(bits):
        t = torch.randint(-(2**63), 2**63 - 1, (B, n, (bits + 63) // 64), generator=g,
                          dtype=torch.int64)
        if bits % 64:
            t[..., -1] &= (1 << (bits % 64)) - 1
        return t.view(torch.uint64).pin_memory()

    acc_h = (rnd(q), rnd(q))
    fresh_h = [(rnd(q), rnd(q)) for _ in range(K)]
    evk = (rnd(2 * q)[0].contiguous().numpy(), rnd(2 * q)[0].contiguous().numpy())
    nph = lambda t: t.numpy()  # noqa: E731
    Lr = (q - K * p.log_p + 63) // 64
    res_h = tuple(torch.empty((B, n, Lr), dtype=torch.uint64).pin_memory() for _ in range(2))
    dl = lambda a: a.download(out=(nph(res_h[0]), nph(res_h[1])))  # noqa: E731

    def uploads(asyn):
        a = ctx.upload((nph(acc_h[0]), nph(acc_h[1])), q, asynchronous=asyn)
        f = [ctx.upload((nph(x[0]), nph(x[1])), q, asynchronous=asyn) for x in fresh_h]
        return a, f

    def compute(a, f):
        for x in f:
            x = ctx.mod_down_dev(x, a.log_q) if x.log_q > a.log_q else x
            a = ctx.he_mul_dev(a, x, evk=evk, evk_id=1)
        return a

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1), (time.perf_counter() - t0) * 1e3, r

    dl(compute(*uploads(False)))  # warm every level
    out = {}
    out["upload_sync_ms"], out["upload_sync_wall_ms"], ops = timed(lambda: uploads(False))
    out["upload_async_ms"], out["upload_async_wall_ms"], _ = timed(lambda: uploads(True))
    out["compute_ms"], out["compute_wall_ms"], _ = timed(lambda: compute(*ops))
    del ops
    out["chain_sync_ms"], out["chain_sync_wall_ms"], _ = timed(
        lambda: dl(compute(*uploads(False))))
    out["chain_async_ms"], out["chain_async_wall_ms"], _ = timed(
        lambda: dl(compute(*uploads(True))))
    # per-operation device times inside one chain (events between calls)
    for asyn in (False, True):
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True)]
        evs[0].record(stream)
        a, f = uploads(asyn)
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append(e)
        for x in f:
            x = ctx.mod_down_dev(x, a.log_q) if x.log_q > a.log_q else x
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append(e)
            a = ctx.he_mul_dev(a, x, evk=evk, evk_id=1)
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append(e)
        dl(a)
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        evs.append(e)
        torch.cuda.synchronize()
        out[f"ops_{'async' if asyn else 'sync'}_ms"] = [round(evs[i].elapsed_time(evs[i + 1]), 2)
                                                       for i in range(len(evs) - 1)]
    out["h2d_gb"] = (K + 1) * 2 * B * n * L * 8 / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
