"""HEA1 files, the parameter JSON and the `hemul` CLI relinked against the
B200 drop-in (proj/core/src/io.cpp:54-208,
proj/tools/hemul.cpp:86-377, exit codes 0/1/2/3).

CPU: the file formats are byte-identical to the reference's writers
(oracle/_ref built with io.cpp) and the CLI's usage / format errors.
GPU: keygen -> encrypt -> mul -> decrypt through the CLI, the product equal
to the reference's he_mul on the same files, and the pinned device loader.
"""
from __future__ import annotations

import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
CLI = ROOT / "paper_2003_04510_b200" / "lib" / "hemul"


def hemul(*args, env=None, timeout=900):
    assert CLI.exists(), "run python -m paper_2003_04510_b200.build"
    e = dict(os.environ)
    e.pop("HEAAN_SEED", None)
    e.update(env or {})
    return subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True,
                          timeout=timeout, env=e)


def read_hea1(path):
    raw = Path(path).read_bytes()
    assert raw[:4] == b"HEA1"
    wb, n, log_q, slots = np.frombuffer(raw[4:20], np.uint32)
    L = (int(log_q) + 63) // 64
    words = np.frombuffer(raw[20:], np.uint64)
    assert words.size == 2 * n * L
    return int(log_q), int(slots), words[:n * L].reshape(n, L), words[n * L:].reshape(n, L)


def test_usage_errors_exit_1(tmp_path):
    assert hemul().returncode == 1
    assert hemul("frobnicate").returncode == 1
    assert hemul("mul", "--params", "x").returncode == 1          # missing required options
    assert hemul("bench", "--radix", "3").returncode == 1
    assert hemul("keygen", "--log-p", "abc").returncode == 1
    assert hemul("cost").returncode == 1


def test_format_errors_exit_3(tmp_path):
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XXXX" + b"\0" * 16)
    params = tmp_path / "params.json"
    params.write_text('{"n": 1024, "log_delta": 30, "log_p": 30, "depth": 4, "log_q_max": 120,'
                      ' "word_bits": 64}')
    r = hemul("mul", "--params", params, "--ct1", bad, "--ct2", bad, "--evk", bad,
              "--out", tmp_path / "o.bin")
    assert r.returncode == 3 and "bad magic" in r.stderr
    (tmp_path / "p2.json").write_text("{not json")
    r = hemul("decrypt", "--params", tmp_path / "p2.json", "--sk", bad, "--ct", bad)
    assert r.returncode == 3 and "bad parameter file" in r.stderr
    assert hemul("keygen", "--out-dir", tmp_path / "missing").returncode == 3


def test_params_json_matches_reference_writer(tmp_path, reference):
    """save_params writes the reference's bytes (nlohmann dump(2) layout)."""
    import ctypes

    fn = reference.lib.ref_save_params
    fn.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    ref_path = tmp_path / "ref.json"
    assert fn(str(ref_path).encode(), 30, 40, 0) == 0
    exe = ROOT / "paper_2003_04510_b200" / "lib" / "dropin_check"
    ours = tmp_path / "ours.json"
    r = subprocess.run([str(exe), "params", "30", "40", "0", str(ours)], capture_output=True,
                       text=True)
    assert r.returncode == 0, r.stderr
    assert ours.read_bytes() == ref_path.read_bytes()
    assert json.loads(ours.read_text())["primes_region2"] > 0


@pytest.mark.gpu
def test_cli_roundtrip_matches_reference(tmp_path, reference):
    """keygen / encrypt / mul / decrypt through the CLI (S-sized ring): the
    product file equals the reference's he_mul on the same ciphertexts, the
    decryption is the slot-wise product, and re-running keygen refuses to
    overwrite (exit 2) unless --force."""
    cfg = ["--log-p", 30, "--depth", 4, "--ring-degree", 11]
    r = hemul("keygen", *cfg, "--out-dir", tmp_path, "--seed", 5)
    assert r.returncode == 0, r.stderr
    assert hemul("keygen", *cfg, "--out-dir", tmp_path).returncode == 2
    assert hemul("keygen", *cfg, "--out-dir", tmp_path, "--force", "--seed", 5).returncode == 0
    P = tmp_path / "params.json"
    r1 = hemul("encrypt", "--params", P, "--pk", tmp_path / "pk.bin", "--out", tmp_path / "a.bin",
               "--values", "0.5,-0.25,0.75,1", "--seed", 3)
    r2 = hemul("encrypt", "--params", P, "--pk", tmp_path / "pk.bin", "--out", tmp_path / "b.bin",
               "--values", "0.5,0.5,-1,0.25", "--seed", 4)
    assert r1.returncode == 0 and r2.returncode == 0, r1.stderr + r2.stderr
    r = hemul("mul", "--params", P, "--ct1", tmp_path / "a.bin", "--ct2", tmp_path / "b.bin",
              "--evk", tmp_path / "evk.bin", "--out", tmp_path / "c.bin")
    assert r.returncode == 0, r.stderr
    q, slots, ca, cb = read_hea1(tmp_path / "c.bin")
    assert q == 90 and slots == 4
    _, _, a_ax, a_bx = read_hea1(tmp_path / "a.bin")
    _, _, b_ax, b_bx = read_hea1(tmp_path / "b.bin")
    _, _, e_ax, e_bx = read_hea1(tmp_path / "evk.bin")
    st, wa, wb = reference.he_mul(30, 4, 11, 120, (a_ax.copy(), a_bx.copy()),
                                  (b_ax.copy(), b_bx.copy()), (e_ax.copy(), e_bx.copy()))
    assert st == 0 and np.array_equal(ca, wa) and np.array_equal(cb, wb)
    r = hemul("decrypt", "--params", P, "--sk", tmp_path / "sk.bin", "--ct", tmp_path / "c.bin")
    assert r.returncode == 0, r.stderr
    got = [complex(re_, im) for re_, im in json.loads(r.stdout)]
    want = [0.25, -0.125, -0.75, 0.25]
    assert max(abs(g - w) for g, w in zip(got, want)) < 1e-3
    # a mul at mismatched moduli is a state error (exit 2)
    r = hemul("mul", "--params", P, "--ct1", tmp_path / "a.bin", "--ct2", tmp_path / "c.bin",
              "--evk", tmp_path / "evk.bin", "--out", tmp_path / "d.bin")
    assert r.returncode == 2 and "moduli differ" in r.stderr
    # bench through the CLI prints the reference's table
    r = hemul("bench", *cfg, "--reps", 2, "--format", "json")
    assert r.returncode == 0, r.stderr


@pytest.mark.gpu
def test_pinned_device_load_save(tmp_path):
    from paper_2003_04510_b200.hemul import Context, make_params

    ctx = Context(make_params(30, 80, 0))
    rng = np.random.default_rng(3)
    n, L = ctx.n, 38
    ax = rng.integers(0, 2**64, (n, L), dtype=np.uint64)
    bx = rng.integers(0, 2**64, (n, L), dtype=np.uint64)
    ax[:, -1] &= np.uint64((1 << 32) - 1)
    bx[:, -1] &= np.uint64((1 << 32) - 1)
    path = tmp_path / "x.bin"
    path.write_bytes(b"HEA1" + np.array([64, n, 2400, 7], np.uint32).tobytes() + ax.tobytes()
                     + bx.tobytes())
    d, slots = ctx.load_dev(str(path))
    assert slots == 7 and d.log_q == 2400
    ga, gb = d.download()
    assert np.array_equal(ga, ax) and np.array_equal(gb, bx)
    ctx.save_dev(d, str(tmp_path / "y.bin"), 7)
    assert (tmp_path / "y.bin").read_bytes() == path.read_bytes()
    (tmp_path / "t.bin").write_bytes(path.read_bytes()[:1000])
    with pytest.raises(Exception, match="truncated"):
        ctx.load_dev(str(tmp_path / "t.bin"))
