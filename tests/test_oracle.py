"""CPU tests: the C restatement oracle (oracle/hemul_oracle.c) pinned against
the reference itself (oracle/_ref, built from /root/reference sources) and
against the committed golden vectors (tests/golden/, made by
tests/golden/gen_golden.py from the reference).

Restates the hot-path reference tests: test_params.cpp:25-59 (primes, roots,
counts), test_ntt.cpp:59-118 (round trip, known answer), test_rns.cpp:21-154
(CRT, iCRT incl. centered lift and negatives, pointwise), test_heaan.cpp:
129-199 (he_mul) and the digest protocol of bench.cpp:35-124.
"""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import limbs, random_poly

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_known_answers_spec(restated):
    # N=4, p=17: [1,0,0,0] -> [1,1,1,1] (any psi)
    tw, itw, ninv = restated.ntt_tables(17, 9, 2)
    out = restated.ntt(np.array([[1, 0, 0, 0]], np.uint64), np.array([17], np.uint64),
                       np.array([9], np.uint64), 2)
    assert out.tolist() == [[1, 1, 1, 1]]
    # CRT of 100 over {17, 19, 23} -> {15, 5, 8}
    r = restated.crt(np.array([[100]], np.uint64), 1, 1, np.array([17, 19, 23], np.uint64))
    assert r.ravel().tolist() == [15, 5, 8]


@pytest.mark.parametrize("region", [1, 2])
@pytest.mark.parametrize("log_n,log_q,log_q_max", [(13, 120, 120), (10, 90, 120), (16, 1200, 1200),
                                                    (17, 2400, 2400), (17, 30 * 41, 2400)])
def test_region_primes_match_reference(region, log_n, log_q, log_q_max, restated, reference):
    a = restated.region_primes(region, log_q, log_q_max, log_n)
    b = reference.level_primes(region, log_q, log_q_max, log_n)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # test_params.cpp:25-51: in (2^57, 2^60), = 1 mod 2n, psi of order 2n
    p = [int(x) for x in a[0]]
    assert all((1 << 57) < x < (1 << 60) and x % (2 << log_n) == 1 for x in p)
    for x, psi in zip(p[:3], a[1][:3]):
        assert pow(int(psi), 1 << log_n, x) == x - 1


def test_prime_counts_paper_point(restated):
    # test_params.cpp:53-59 — np = 42 / 63 at logq = 1200 (w64)
    assert len(restated.region_primes(1, 1200, 1200, 16)[0]) == 42
    assert len(restated.region_primes(2, 1200, 1200, 16)[0]) == 63
    assert len(restated.region_primes(1, 2400, 2400, 17)[0]) == 84
    assert len(restated.region_primes(2, 2400, 2400, 17)[0]) == 125


@pytest.mark.parametrize("region", [1, 2])
def test_stages_match_reference(region, restated, reference):
    log_n, log_q, qmax = 10, 120, 120
    primes, roots = restated.region_primes(region, log_q, qmax, log_n)
    n, np_ = 1 << log_n, len(primes)
    rng = np.random.default_rng(5)
    bits_b = log_q if region == 1 else 2 * qmax
    a = random_poly(rng, n, log_q)
    b = random_poly(rng, n, bits_b)
    # pm_prepare = CRT + NTT (polymul.cpp:7-20)
    fa = restated.ntt(restated.crt(a, n, limbs(log_q), primes), primes, roots, log_n)
    fb = restated.ntt(restated.crt(b, n, limbs(bits_b), primes), primes, roots, log_n)
    assert np.array_equal(fa, reference.prepare(region, log_q, qmax, log_n, log_q, a, np_))
    assert np.array_equal(fb, reference.prepare(region, log_q, qmax, log_n, bits_b, b, np_))
    prod = restated.pointwise(fa, fb, primes, n)
    assert np.array_equal(prod, reference.pointwise(region, log_q, qmax, log_n, fa, fb))
    tbits = log_q if region == 1 else log_q + qmax
    inv = restated.ntt(prod, primes, roots, log_n, inverse=True)
    assert np.array_equal(restated.icrt(inv, n, primes, tbits),
                          reference.finish(region, log_q, qmax, log_n, prod, tbits))


def test_icrt_centered_lift_edges(restated, reference):
    """test_rns.cpp:91-133: values near P/2, negatives, zero."""
    log_n, log_q, qmax = 10, 120, 120
    primes, _ = restated.region_primes(1, log_q, qmax, log_n)
    n = 1 << log_n
    rng = np.random.default_rng(8)
    x = np.stack([rng.integers(0, int(p), size=n, dtype=np.uint64) for p in primes])
    x[:, 0] = 0
    x[:, 1] = primes - np.uint64(1)  # -1
    x[:, 2] = 1
    got = restated.icrt(x, n, primes, log_q)
    want = reference.finish(1, log_q, qmax, log_n, x, log_q, skip_intt=True)
    assert np.array_equal(got, want)
    assert got[0].tolist() == [0, 0]
    assert got[1].tolist() == [(1 << 64) - 1, (1 << (log_q - 64)) - 1]  # -1 mod 2^120


def test_ntt_round_trip_exhaustive_small(restated):
    """test_ntt.cpp:59-104 in spirit: all 17^4 inputs at N=4, p=17."""
    p = np.array([17], np.uint64)
    psi = np.array([9], np.uint64)
    xs = np.array(np.meshgrid(*[np.arange(17)] * 4, indexing="ij")).reshape(4, -1).T
    xs = np.ascontiguousarray(xs, dtype=np.uint64)
    fwd = restated.ntt(xs, p, psi, 2)
    back = restated.ntt(fwd, p, psi, 2, inverse=True)
    assert np.array_equal(back, xs)


@pytest.mark.parametrize("cfg", [(30, 4, 10), (30, 6, 11), (20, 4, 10)])
def test_he_mul_matches_reference_every_level(cfg, restated, reference):
    log_n, n, qmax = reference.make_params(*cfg)
    rng = np.random.default_rng(sum(cfg))
    evk = (random_poly(rng, n, 2 * qmax), random_poly(rng, n, 2 * qmax))
    for log_q in range(qmax, 2 * cfg[0] - 1, -cfg[0]):
        c1 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        c2 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        st1, a1, b1 = restated.he_mul(log_n, cfg[0], qmax, log_q, c1, c2, evk)
        st2, a2, b2 = reference.he_mul(*cfg, log_q, c1, c2, evk)
        assert st1 == st2 == 0
        assert np.array_equal(a1, a2) and np.array_equal(b1, b2)


def test_he_mul_error_kinds(restated, reference):
    log_n, n, qmax = reference.make_params(30, 4, 10)
    z = np.zeros((n, 2), np.uint64)
    e = np.zeros((n, 4), np.uint64)
    assert restated.he_mul(log_n, 30, qmax, 120, (z, z), (z, z), (e, e), c2_log_q=90)[0] == 2
    assert reference.he_mul(30, 4, 10, 120, (z, z), (z, z), (e, e), c2_log_q=90)[0] == 2
    z1 = np.zeros((n, 1), np.uint64)
    assert restated.he_mul(log_n, 30, qmax, 30, (z1, z1), (z1, z1), (e, e))[0] == 3
    assert reference.he_mul(30, 4, 10, 30, (z1, z1), (z1, z1), (e, e))[0] == 3


def test_golden_s_bench_fixture(restated):
    """The committed S fixture (reference output) reproduces with the oracle,
    and its digest is the reference's."""
    g = np.load(GOLDEN / "s_bench.npz")
    d = json.loads((GOLDEN / "digests.json").read_text())["S"]
    q = int(g["log_q"])
    st, oa, ob = restated.he_mul(13, 30, q, q, (g["c1ax"], g["c1bx"]), (g["c2ax"], g["c2bx"]),
                                 (g["evkax"], g["evkbx"]))
    assert st == 0
    assert np.array_equal(oa, g["outax"]) and np.array_equal(ob, g["outbx"])
    assert f"{restated.digest(q - 30, 1 << 13, oa, ob):016x}" == d["digest"]


def test_golden_small_random_fixture(restated):
    g = np.load(GOLDEN / "small_random.npz")
    log_p, depth, log_n = (int(v) for v in g["params"])
    evk = (g["evkax"], g["evkbx"])
    for lvl in (0, 1):
        q = int(g[f"log_q_{lvl}"])
        st, oa, ob = restated.he_mul(log_n, log_p, log_p * depth, q,
                                     (g[f"c1ax_{lvl}"], g[f"c1bx_{lvl}"]),
                                     (g[f"c2ax_{lvl}"], g[f"c2bx_{lvl}"]), evk)
        assert st == 0
        assert np.array_equal(oa, g[f"outax_{lvl}"]) and np.array_equal(ob, g[f"outbx_{lvl}"])


def test_golden_digests_reproduce_with_reference(reference):
    """Seed-7 bench protocol digests of the small configs (M and X take
    minutes on CPU; they are checked on the GPU box against the same file)."""
    golden = json.loads((GOLDEN / "digests.json").read_text())
    for name in ("S", "logN13_logQ300"):
        dig, _ = reference.run_bench(*golden[name]["params"], seed=7, reps=1)
        assert f"{dig:016x}" == golden[name]["digest"]
    assert golden["M"]["digest"] == "cf360cab57109023"
    assert golden["X"]["digest"] == "1293cdbbebaf5349"
