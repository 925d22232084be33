"""The multi-rank bench path through the real CUDA library on one GPU.

bench.py under torchrun with two ranks sharing cuda:0 (gloo process group;
the driver's scaling runs use the same code with NCCL, one GPU per rank):
every rank builds its own level tables and evk forms, runs its own block of
HE Muls, the slowest rank's device time sets `value`, and rank 0 gathers one
digest per rank after the timed region. Each gathered digest must equal the
digest of the same inputs (bench.make_inputs, seed 1000 + rank) computed in
this process by a single Context.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_ranks_one_gpu_bench_path():
    steps, warmup, batch = 3, 3, 4
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(ROOT / "bench.py"),
           "--gpus", "2", "--config", "S", "--batch", str(batch), "--steps", str(steps),
           "--warmup", str(warmup), "--dist-backend", "gloo", "--one-device",
           "--no-cpu-baseline", "--chain", "0", "--latency-reps", "1"]
    env = dict(os.environ, PYTHONPATH=str(ROOT))
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["global_batch"] == 2 * batch
    assert d["config"]["dist_backend"] == "gloo"
    # value = all ranks' HE Muls / the slowest rank's device time
    assert d["value"] == pytest.approx(2 * batch * steps / (d["ms_per_step"] * steps / 1e3),
                                       rel=1e-6)
    assert d["gpu_launches"] > 0
    assert len(d["digests"]) == 2 and d["digests"][0] != d["digests"][1]

    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2003_04510_b200.hemul import Context, ciphertext_digest, make_params

    p = make_params(*bench.CONFIGS["S"])
    q = p.log_q_max
    ctx = Context(p, device=0)
    for rank, want in enumerate(d["digests"]):
        c1, c2, evk = bench.make_inputs(p.n, q, batch, seed=1000 + rank)
        oa, ob = ctx.he_mul((c1[0][:1], c1[1][:1]), (c2[0][:1], c2[1][:1]), q, evk=evk,
                            evk_id=0)
        got = ciphertext_digest(q - p.log_p, oa[0].cpu().numpy(), ob[0].cpu().numpy())
        assert f"{got:016x}" == want, rank
    ctx.close()
