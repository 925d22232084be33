"""CPU: the numpy residue helpers of tests/modmath.py (the expected values of
the 30-bit-basis stage tests) pinned against the C restatement of the
reference's CRT / NTT / pointwise / iCRT (oracle/hemul_oracle.c) on 30-bit
primes p = 1 mod 2n."""
from __future__ import annotations

import numpy as np

import modmath as mm
from oracle_lib import limbs, random_poly


def _primes30(count: int, log_n: int) -> list[int]:
    two_n = 2 << log_n
    out = []
    c = (1 << 30) - 1
    c -= (c - 1) % two_n
    while len(out) < count:
        if all(pow(a, c - 1, c) == 1 for a in (2, 3, 5, 7, 11, 13)):
            out.append(c)
        c -= two_n
    return out


def test_residues_match_oracle_crt(restated):
    rng = np.random.default_rng(1)
    n, bits = 256, 300
    a = random_poly(rng, n, bits)
    primes = np.array(_primes30(7, 8), np.uint64)
    want = restated.crt(a, n, limbs(bits), primes)
    got = mm.residues(mm.poly_ints(a), primes)
    assert np.array_equal(got, want)


def test_negacyclic_matches_oracle_ntt_pipeline(restated):
    rng = np.random.default_rng(2)
    log_n = 7
    n = 1 << log_n
    primes = _primes30(3, log_n)
    roots = [mm.root_2n(p, n) for p in primes]
    a = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
    b = np.stack([rng.integers(0, p, n, dtype=np.uint64) for p in primes])
    fa = restated.ntt(a, np.array(primes, np.uint64), roots, log_n)
    fb = restated.ntt(b, np.array(primes, np.uint64), roots, log_n)
    prod = np.stack([fa[j] * fb[j] % np.uint64(p) for j, p in enumerate(primes)])
    want = restated.ntt(prod, np.array(primes, np.uint64), roots, log_n, inverse=True)
    assert np.array_equal(mm.negacyclic(a, b, primes), want)


def test_centred_lift_matches_oracle_icrt(restated):
    rng = np.random.default_rng(3)
    n = 64
    primes = np.array(_primes30(5, 6), np.uint64)
    P = 1
    for p in primes:
        P *= int(p)
    vals = [int(rng.integers(0, 1 << 62)) * int(rng.integers(0, 1 << 62)) % P - P // 2
            for _ in range(n)]
    res = mm.residues([v % P for v in vals], primes)
    assert mm.centred_lift(res, primes) == [v if v != -(P // 2) else v for v in vals]
    T = 200
    want = restated.icrt(res, n, primes, T)
    assert np.array_equal(mm.ints_poly(mm.centred_lift(res, primes), T), want)
