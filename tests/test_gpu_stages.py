"""Stage-level parity on the GPU: every kernel against the oracles on the same
level tables (test_ntt.cpp / test_rns.cpp / test_polymul.cpp restated).

Residues must be bit-identical: they are canonical, so the reference's Shoup
variants, radices and accumulation strategies all produce exactly these
values (test_ntt.cpp:120-165, test_rns.cpp:21-45, test_polymul.cpp:91-117).
"""
from __future__ import annotations

import numpy as np
import pytest

from oracle_lib import limbs, random_poly

pytestmark = pytest.mark.gpu

# (log_p, depth, log_n_override): S and two small rings; M runs in the
# dedicated slow test below.
CONFIGS = [(30, 4, 13), (30, 4, 10), (30, 6, 12)]


def _ctx(cfg):
    from paper_2003_04510_b200.hemul import Context, make_params

    return Context(make_params(*cfg))


def _residues(rng, primes, n, rows):
    out = np.empty((rows, n), np.uint64)
    for r in range(rows):
        out[r] = rng.integers(0, int(primes[r % len(primes)]), size=n, dtype=np.uint64)
    return out


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("region", [1, 2])
def test_level_primes_match_reference_rules(cfg, region, restated):
    ctx = _ctx(cfg)
    p = ctx.params
    for log_q in (p.log_q_max, p.log_q_max - p.log_p):
        want, _ = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
        got = ctx.level_primes(log_q, region)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("region", [1, 2])
def test_ntt_forward_inverse_bit_exact(cfg, region, restated):
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max
    primes, roots = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
    rng = np.random.default_rng(3)  # bench_ntt.cpp:17-20 style inputs
    rows = 2 * len(primes) + 1       # batch of two transforms + one ragged row
    x = _residues(rng, primes, p.n, rows)
    want = restated.ntt(x, primes, roots, p.log_n)
    got = x.copy()
    ctx.ntt(got, log_q, region)
    assert np.array_equal(got, want)
    back = got.copy()
    ctx.ntt(back, log_q, region, inverse=True)
    assert np.array_equal(back, x)  # round trip (test_ntt.cpp:59-104)
    want_inv = restated.ntt(want, primes, roots, p.log_n, inverse=True)
    assert np.array_equal(want_inv, x)


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("region,which", [(1, "q"), (2, "q"), (2, "evk")])
def test_crt_bit_exact(cfg, region, which, restated):
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max - p.log_p
    bits = log_q if which == "q" else 2 * p.log_q_max
    primes, _ = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
    rng = np.random.default_rng(11)
    poly = random_poly(rng, p.n, bits)
    poly[0] = 0                                     # zero coefficient
    poly[1] = np.uint64(0xFFFFFFFFFFFFFFFF)         # all-ones limbs
    if bits % 64:
        poly[1, -1] = np.uint64((1 << (bits % 64)) - 1)
    want = restated.crt(poly, p.n, limbs(bits), primes)
    got = ctx.crt(poly, log_q, region, bits)
    assert np.array_equal(got, want)
    # batched call = per-poly calls
    two = np.stack([poly, poly[::-1].copy()])
    got2 = ctx.crt(two, log_q, region, bits)
    assert np.array_equal(got2[0], want)
    assert np.array_equal(got2[1], restated.crt(two[1], p.n, limbs(bits), primes))


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("region", [1, 2])
def test_pointwise_bit_exact(cfg, region, restated):
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max
    primes, _ = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
    rng = np.random.default_rng(5)
    a = _residues(rng, primes, p.n, len(primes))
    b = _residues(rng, primes, p.n, len(primes))
    a[:, 0] = primes - np.uint64(1)                 # (p-1)^2 edge
    b[:, 0] = primes - np.uint64(1)
    want = restated.pointwise(a, b, primes, p.n)
    assert np.array_equal(ctx.pointwise(a, b, log_q, region), want)


@pytest.mark.parametrize("cfg", CONFIGS)
@pytest.mark.parametrize("region", [1, 2])
def test_icrt_of_products_bit_exact(cfg, region, restated):
    """pm_finish on genuine products (the domain he_mul feeds the iCRT)."""
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max
    primes, roots = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
    rng = np.random.default_rng(17)
    bits_b = log_q if region == 1 else 2 * p.log_q_max
    a = random_poly(rng, p.n, log_q)
    b = random_poly(rng, p.n, bits_b)
    fa = restated.ntt(restated.crt(a, p.n, limbs(log_q), primes), primes, roots, p.log_n)
    fb = restated.ntt(restated.crt(b, p.n, limbs(bits_b), primes), primes, roots, p.log_n)
    prod = restated.ntt(restated.pointwise(fa, fb, primes, p.n), primes, roots, p.log_n,
                        inverse=True)
    tbits = log_q if region == 1 else log_q + p.log_q_max
    want = restated.icrt(prod, p.n, primes, tbits)
    assert np.array_equal(ctx.icrt(prod, log_q, region), want)


@pytest.mark.parametrize("cfg", CONFIGS[:1])
@pytest.mark.parametrize("region", [1, 2])
def test_icrt_arbitrary_residues_exact_fallback(cfg, region, restated):
    """Uniform residues put |v| anywhere in (-P/2, P/2): half the coefficients
    take the exact fix-up path (rns.cpp:148-169 centered lift near P/2)."""
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max
    primes, _ = restated.region_primes(region, log_q, p.log_q_max, p.log_n)
    rng = np.random.default_rng(23)
    x = _residues(rng, primes, p.n, len(primes))
    x[:, 0] = 0                                      # v = 0
    x[:, 1] = primes - np.uint64(1)                  # v = -1
    tbits = log_q if region == 1 else log_q + p.log_q_max
    want = restated.icrt(x, p.n, primes, tbits)
    assert np.array_equal(ctx.icrt(x, log_q, region), want)


@pytest.mark.slow
@pytest.mark.parametrize("region", [1, 2])
def test_stages_paper_point_M(region, reference):
    """N=2^16, logQ=1200 (np 42/63): prepare / finish vs the reference's own
    pm_prepare / pm_finish on its tables."""
    cfg = (30, 40, 0)
    ctx = _ctx(cfg)
    p = ctx.params
    log_q = p.log_q_max
    np_ = len(ctx.level_primes(log_q, region))
    rng = np.random.default_rng(29)
    bits_b = log_q if region == 1 else 2 * p.log_q_max
    a = random_poly(rng, p.n, log_q)
    b = random_poly(rng, p.n, bits_b)
    fa_ref = reference.prepare(region, log_q, p.log_q_max, p.log_n, log_q, a, np_)
    fb_ref = reference.prepare(region, log_q, p.log_q_max, p.log_n, bits_b, b, np_)
    fa = ctx.crt(a, log_q, region, log_q)
    ctx.ntt(fa, log_q, region)
    assert np.array_equal(fa, fa_ref)
    fb = ctx.crt(b, log_q, region, bits_b)
    ctx.ntt(fb, log_q, region)
    assert np.array_equal(fb, fb_ref)
    prod = ctx.pointwise(fa, fb, log_q, region)
    assert np.array_equal(prod, reference.pointwise(region, log_q, p.log_q_max, p.log_n,
                                                    fa_ref, fb_ref))
    tbits = log_q if region == 1 else log_q + p.log_q_max
    want = reference.finish(region, log_q, p.log_q_max, p.log_n, prod, tbits)
    ctx.ntt(prod, log_q, region, inverse=True)
    assert np.array_equal(ctx.icrt(prod, log_q, region), want)
