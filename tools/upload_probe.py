"""Host-side cost of one asynchronous upload (is the call really async?)."""
import sys, time, json
from pathlib import Path
import torch
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2003_04510_b200.hemul import Context, make_params  # noqa: E402

p = make_params(30, 80, 0)
q, n = p.log_q_max, p.n
ctx = Context(p)
stream = torch.cuda.Stream(); torch.cuda.set_stream(stream); ctx.set_stream(stream.cuda_stream)
B = 8
h = torch.zeros((B, n, 38), dtype=torch.int64).view(torch.uint64).pin_memory()
d = torch.empty((B, n, 38), dtype=torch.uint64, device="cuda")
out = {"is_pinned": bool(h.is_pinned())}
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); d.copy_(h, non_blocking=True)
    out[f"torch_copy_wall_ms_{rep}"] = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    t0 = time.perf_counter(); x = ctx.upload((h.numpy(), h.numpy()), q, asynchronous=True)
    out[f"upload_async_wall_ms_{rep}"] = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    t0 = time.perf_counter(); y = ctx.upload((h.numpy(), h.numpy()), q, asynchronous=False)
    out[f"upload_sync_wall_ms_{rep}"] = (time.perf_counter() - t0) * 1e3
    del x, y
print(json.dumps(out))
