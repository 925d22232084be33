"""The C++ drop-in API (include/hemul/*.hpp, namespace hemul) as a user of
the reference would consume it: tests/cpp/dropin_check.cpp is compiled
against libhemul_gpu.so with the reference's type and function names.

CPU: the host-side keygen / encode / encrypt reproduce the reference's
     seed-7 transcript bit for bit (bench.cpp:60-67).
GPU: run_he_mul_bench's digest equals the reference's golden digest; the
     multiplication ladder decrypts correctly (test_heaan.cpp:143-167); the
     error kinds match (test_heaan.cpp:169-182).
"""
from __future__ import annotations

import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
BIN = ROOT / "paper_2003_04510_b200" / "lib" / "dropin_check"
GOLDEN = Path(__file__).resolve().parent / "golden"


def _run(*args, timeout=600):
    assert BIN.exists(), "run python -m paper_2003_04510_b200.build"
    return subprocess.run([str(BIN), *map(str, args)], capture_output=True, text=True,
                          timeout=timeout)


@pytest.mark.parametrize("cfg", [(30, 4, 13), (30, 10, 0), (30, 6, 11)])
def test_host_keys_and_ciphertexts_match_reference(cfg, tmp_path, reference):
    res = _run("keys", *cfg, 7, str(tmp_path) + "/")
    assert res.returncode == 0, res.stderr
    want = reference.bench_inputs(*cfg, seed=7)
    for name, arr in (("c1ax", want["c1"][0]), ("c1bx", want["c1"][1]), ("c2ax", want["c2"][0]),
                      ("c2bx", want["c2"][1]), ("evkax", want["evk"][0]),
                      ("evkbx", want["evk"][1])):
        got = np.fromfile(tmp_path / name, dtype=np.uint64).reshape(arr.shape)
        assert np.array_equal(got, arr), name


def test_host_keys_match_committed_fixture(tmp_path):
    """Same check without the reference build: the S fixture's inputs."""
    g = np.load(GOLDEN / "s_bench.npz")
    res = _run("keys", 30, 4, 13, 7, str(tmp_path) + "/")
    assert res.returncode == 0, res.stderr
    for name in ("c1ax", "c1bx", "c2ax", "c2bx", "evkax", "evkbx"):
        got = np.fromfile(tmp_path / name, dtype=np.uint64).reshape(g[name].shape)
        assert np.array_equal(got, g[name]), name


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["S", "logN13_logQ300", "M"])
def test_run_he_mul_bench_digest(name):
    d = json.loads((GOLDEN / "digests.json").read_text())[name]
    p = d["params"]
    res = _run("bench", p[0], p[1], p[2], 7, 2, timeout=900)
    assert res.returncode == 0, res.stderr
    assert re.search(r"digest ([0-9a-f]+)", res.stdout).group(1) == d["digest"]


@pytest.mark.gpu
def test_ladder_decrypts():
    res = _run("ladder", 30, 6, 11, 7)
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.gpu
def test_error_kinds():
    res = _run("errors")
    assert res.returncode == 0, res.stdout + res.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", [(30, 6, 11), (30, 10, 13)])
def test_ladder_device_resident(cfg):
    """Scheme::upload / he_mul / mod_down / download on DeviceCiphertext: the
    ladder (test_heaan.cpp:143-167) with the accumulator kept in HBM equals the
    host-API ladder bit for bit at every step and decrypts correctly."""
    res = _run("ladder_dev", *cfg, 7)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "mismatches 0" in res.stdout
