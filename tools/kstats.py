"""Per-kernel-class device times of a few batched HE Muls at X (no checks):
a quick tool for kernel experiments.  python tools/kstats.py [--steps 3]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2003_04510_b200.hemul import Context, make_params  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--batch", type=int, default=8)
a = ap.parse_args()
p = make_params(30, 80, 0)
ctx = Context(p)
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
ctx.set_stream(st.cuda_stream)
q, n, B = p.log_q_max, p.n, a.batch
L = (q + 63) // 64


def rp(b, bits):
    t = torch.randint(-(2**63), 2**63 - 1, (b, n, (bits + 63) // 64), device="cuda", dtype=torch.int64)
    if bits % 64:
        t[..., -1] &= (1 << (bits % 64)) - 1
    return t.view(torch.uint64)


c1, c2 = (rp(B, q), rp(B, q)), (rp(B, q), rp(B, q))
evk = (rp(1, 2 * q)[0].contiguous(), rp(1, 2 * q)[0].contiguous())
Lo = (q - p.log_p + 63) // 64
out = (torch.empty((B, n, Lo), dtype=torch.uint64, device="cuda"),
       torch.empty((B, n, Lo), dtype=torch.uint64, device="cuda"))
ctx.warm_level(q, evk, evk_id=1)
for _ in range(2):
    ctx.he_mul(c1, c2, q, evk=evk, evk_id=1, out=out)
torch.cuda.synchronize()
ctx.enable_stage_timing(True)
ctx.reset_stats()
for _ in range(a.steps):
    ctx.he_mul(c1, c2, q, evk=evk, evk_id=1, out=out)
torch.cuda.synchronize()
ks = ctx.kernel_stats()
print({k: round(v[0] / a.steps, 3) for k, v in ks.items() if v[0] > 0})
