"""Residue-level parity of the hot-path kernels of the 30-bit basis, stage by
stage, inside the real he_mul pipeline (hemul_gpu_he_mul_trace).

The stage entry points (test_gpu_stages.py) run the reference's w64 primes;
he_mul runs the B200 basis (30-bit primes, split region 1) through different
kernels: crt_tc.cu (or crt.cu with the IMAD engine), ntt_col.cu, ntt_blk.cu
(middle pass fused with the tensor / evk products), bigint_tc.cu (iCRT of d2
and the fused finisher). Each checkpoint is compared with the reference's
algebra restated in tests/modmath.py (itself pinned to the C restatement by
test_modmath.py):

  CRT1   crt_forward of the eight h-bit halves          rns.cpp:43-106
  PROD1  iNTT(NTT(.) . NTT(.)) split tensor products     polymul.cpp:22-37, heaan.cpp:372-394
  D2     exact centred iCRT of d2 mod 2^log_q            rns.cpp:132-190
  CRT2   ModUp: crt_forward of d2 into region 2          heaan.cpp:398
  PROD2  evk products d2 evk.ax, d2 evk.bx               heaan.cpp:399-400
  final  he_mul against the C restatement                heaan.cpp:339-410

Table shapes (split point, CRT column tiles, iCRT / finisher byte windows)
change with log_q, so every config walks several ladder levels, and the
engine actually used at each level is asserted (no silent fallback).
"""
from __future__ import annotations

import numpy as np
import pytest

import modmath as mm
from oracle_lib import random_poly

pytestmark = pytest.mark.gpu

# (log_p, depth, log_n_override) and the levels walked: paper log_q ranges
# (X: 2400, M: 1200, logN15 row: 600) at small ring degrees
LADDERS = [
    ((30, 80, 12), [2400, 1800, 1230, 600, 300, 90, 60]),
    ((30, 40, 12), [1200, 870, 450, 60]),
    ((30, 20, 13), [600, 330, 60]),
    # paper ring degrees (small log_q): the half-warp column pass and the
    # S = 8 middle pass run only at log N >= 15
    ((30, 4, 16), [120, 60]),
    ((30, 4, 17), [120]),
]


def _ctx(cfg, tc, transposed=None):
    from paper_2003_04510_b200.hemul import Context, make_params

    ctx = Context(make_params(*cfg))
    ctx.set_basis(32)
    ctx.set_tensor_cores(tc)
    if transposed is not None:
        ctx.set_transposed(transposed)
    return ctx


def _natural(rows, log_n, S):
    """Column-major RNS rows (HEMUL_INFO_T_PASS_A = S: position x 2^S + y holds
    coefficient y n / 2^S + x) back in coefficient order."""
    if not S:
        return rows
    r = rows.reshape(rows.shape[0], 1 << (log_n - S), 1 << S)
    return np.ascontiguousarray(r.transpose(0, 2, 1)).reshape(rows.shape[0], 1 << log_n)


def _expected(ctx, info, log_q, c1, c2, evk):
    h = info["split_h"]
    p1 = ctx.level_primes(log_q, -1)
    p2 = ctx.level_primes(log_q, -2)
    assert len(p1) == info["np1"] and len(p2) == info["np2"]
    n = ctx.n
    mask = (1 << h) - 1
    fields = []
    for poly in (c1[0], c1[1], c2[0], c2[1]):  # ax1 bx1 ax2 bx2
        v = mm.poly_ints(poly)
        fields += [[x & mask for x in v], [x >> h for x in v]]
    crt1 = [mm.residues(f, p1) for f in fields]
    plan1 = mm.NttPlan(p1, n)
    P1 = plan1.P
    F = [plan1.fwd(r) for r in crt1]
    x1, X1, y1, Y1, x2, X2, y2, Y2 = F
    sums = [x1 * x2 % P1, (x1 * X2 + X1 * x2) % P1, y1 * y2 % P1, (y1 * Y2 + Y1 * y2) % P1,
            (x1 * y2 + x2 * y1) % P1, (x1 * Y2 % P1 + X1 * y2 % P1 + x2 * Y1 % P1 + X2 * y1) % P1]
    prod1 = [plan1.inv(s) for s in sums]
    c0 = mm.centred_lift(prod1[0], p1)
    ch = mm.centred_lift(prod1[1], p1)
    q = (1 << log_q) - 1
    d2 = [(a + (b << h)) & q for a, b in zip(c0, ch)]
    crt2 = mm.residues(d2, p2)
    plan2 = mm.NttPlan(p2, n)
    fd2 = plan2.fwd(crt2)
    # the 30-bit basis takes the key mod 2^(log_q + log_Q) (context.cu evk_forms)
    kmask = (1 << (log_q + ctx.params.log_q_max)) - 1
    prod2 = [plan2.inv(fd2 * plan2.fwd(mm.residues([x & kmask for x in mm.poly_ints(e)], p2))
                       % plan2.P) for e in evk]
    return {"p1": p1, "p2": p2, "crt1": crt1, "prod1": prod1, "d2": mm.ints_poly(d2, log_q),
            "crt2": crt2, "prod2": prod2}


def _check_rows(got, want_slots, primes, t_form):
    """got: (slots * np, n) device residues (lazy ranges allowed); want: list of
    (np, n) canonical residues."""
    P = np.asarray(primes, np.uint64)[:, None]
    hinv = mm.crt_hat_inverse(primes)[:, None] if t_form else None
    npr = len(primes)
    assert got.shape[0] == len(want_slots) * npr
    for s, want in enumerate(want_slots):
        g = got[s * npr:(s + 1) * npr].astype(np.uint64)
        assert int(g.max()) < 4 * int(P.max()), "residue outside the lazy range"
        w = want * hinv % P if t_form else want
        bad = np.argwhere(g % P != w)
        assert bad.size == 0, f"slot {s}: {len(bad)} residues differ, first (prime, coeff) {bad[0]}"


@pytest.mark.parametrize("tc,trn", [(True, True), (True, False), (False, False)],
                         ids=["tc", "tc-natural", "imad"])
@pytest.mark.parametrize("cfg,levels", LADDERS, ids=["X_logQ@N4096", "M_logQ@N4096",
                                                     "logQ600@N8192", "logQ120@N65536",
                                                     "logQ120@N131072"])
def test_stage_checkpoints_along_the_ladder(cfg, levels, tc, trn, restated):
    if not trn and tc and cfg[2] < 15:
        pytest.skip("the layouts differ only at log N >= 15")
    ctx = _ctx(cfg, tc, trn)
    p = ctx.params
    rng = np.random.default_rng(cfg[1] + 7 * tc)
    evk = (random_poly(rng, p.n, 2 * p.log_q_max), random_poly(rng, p.n, 2 * p.log_q_max))
    for log_q in levels:
        info = ctx.engine_info(log_q)
        assert info["word"] == 32 and info["split_h"] > 0
        assert info["fused_mid"] == 1 and info["blk_mont"] == 1
        if tc:
            # the tensor-core engine must really run at every level (no
            # silent IMAD fallback from a table that does not fit)
            assert info["crt1_tc"] and info["crt2_tc"] and info["big_tc"], (log_q, info)
        c1 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        c2 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        want = _expected(ctx, info, log_q, c1, c2, evk)
        t_form = bool(info["big_tc"])
        S = info["t_pass_a"]
        assert bool(S) == (tc and trn and cfg[2] >= 15), info
        tr = {k: ctx.he_mul_trace(c1, c2, log_q, k, evk=evk)
              for k in ("crt1", "prod1", "d2", "crt2", "prod2")}
        for k in ("crt1", "prod1", "crt2", "prod2"):
            tr[k] = _natural(tr[k], p.log_n, S)
        _check_rows(tr["crt1"], want["crt1"], want["p1"], False)
        _check_rows(tr["prod1"], want["prod1"], want["p1"], t_form)
        assert np.array_equal(tr["d2"].reshape(p.n, -1), want["d2"]), log_q
        _check_rows(tr["crt2"], [want["crt2"]], want["p2"], False)
        _check_rows(tr["prod2"], want["prod2"], want["p2"], t_form)
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, p.log_q_max, log_q, c1, c2, evk)
        assert st == 0
        oa, ob = ctx.he_mul(c1, c2, log_q, evk=evk)
        assert np.array_equal(oa, wa) and np.array_equal(ob, wb), log_q
    ctx.close()


def test_engine_info_levels_at_paper_scale():
    """At N=2^17 / logQ=2400 every ladder level runs the tensor-core engine
    (the iCRT / finisher tables change width with log_q)."""
    ctx = _ctx((30, 80, 0), True)
    for log_q in range(2400, 59, -60):
        info = ctx.engine_info(log_q)
        assert info["word"] == 32
        assert info["crt1_tc"] and info["crt2_tc"] and info["big_tc"], (log_q, info)
    ctx.close()


@pytest.mark.slow
def test_every_level_of_the_logQ2400_ladder(restated):
    """he_mul at all 79 levels of logQ = 2400 (N = 4096) in both engines of the
    30-bit basis against the C restatement: every split point / byte-window
    shape the X ladder produces."""
    cfg = (30, 80, 12)
    ctxs = {tc: _ctx(cfg, tc) for tc in (True, False)}
    p = ctxs[True].params
    rng = np.random.default_rng(2400)
    evk = (random_poly(rng, p.n, 2 * p.log_q_max), random_poly(rng, p.n, 2 * p.log_q_max))
    for log_q in range(p.log_q_max, 2 * p.log_p - 1, -p.log_p):
        c1 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        c2 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, p.log_q_max, log_q, c1, c2, evk)
        assert st == 0
        for tc, ctx in ctxs.items():
            if tc:
                info = ctx.engine_info(log_q)
                assert info["crt1_tc"] and info["crt2_tc"] and info["big_tc"], (log_q, info)
            oa, ob = ctx.he_mul(c1, c2, log_q, evk=evk)
            assert np.array_equal(oa, wa) and np.array_equal(ob, wb), (log_q, tc)
    for ctx in ctxs.values():
        ctx.close()


@pytest.mark.parametrize("log_n", [12, 15, 16, 17])
def test_ntt32_rows_vs_restated(log_n, restated):
    """hemul_gpu_ntt32: the 30-bit column kernels (ntt_col.cu: warp form at
    S = 7, half-warp form at S >= 8) + pass B, residue for residue against the
    C restatement's ntt_forward / ntt_inverse (ntt.cpp:59-137, 153-197) with
    the same primes and min-root rule; lazy GPU outputs compared mod p, and
    the inverse of the GPU forward output returns the input exactly."""
    import torch

    ctx = _ctx((30, 10, log_n), True)
    q = ctx.params.log_q_max
    primes = ctx.level_primes(q, -2)
    npr = min(5, len(primes))
    ps = primes[:npr]
    n = 1 << log_n
    rng = np.random.default_rng(log_n)
    x = (rng.integers(0, 2**62, size=(2 * npr, n), dtype=np.uint64)
         % np.tile(ps, 2).astype(np.uint64)[:, None])
    roots = [mm.root_2n(int(p), n) for p in ps]
    P = np.tile(ps, 2).astype(np.uint64)[:, None]
    dev = torch.from_numpy(x.astype(np.int32)).cuda()
    ctx.ntt32(dev, q, 2, nprimes=npr)
    fwd = dev.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert int(fwd.max()) < 4 * int(P.max())
    want = restated.ntt(x, ps, roots, log_n)
    assert np.array_equal(fwd % P, want % P)
    ctx.ntt32(dev, q, 2, inverse=True, nprimes=npr)
    back = dev.cpu().numpy().view(np.uint32).astype(np.uint64)
    assert np.array_equal(back, x)
    want_inv = restated.ntt(x, ps, roots, log_n, inverse=True)
    dev = torch.from_numpy(x.astype(np.int32)).cuda()
    ctx.ntt32(dev, q, 2, inverse=True, nprimes=npr)
    assert np.array_equal(dev.cpu().numpy().view(np.uint32).astype(np.uint64) % P, want_inv % P)
    ctx.close()


@pytest.mark.parametrize("log_n", [12, 17])
def test_device_twiddles_match_rule(log_n):
    """The 30-bit basis twiddle tables built on the device (tables.cu) equal
    make_ntt_tables' rule (params.cpp:151-180): tw[rev(i)] = psi^i,
    itw[rev(i)] = psi^-i, psi the smallest-c primitive 2n-th root, Shoup
    quotient floor(w 2^32 / p) — for the first, a middle and the last prime
    of both regions."""
    ctx = _ctx((30, 80, log_n), True)
    q = ctx.params.log_q_max
    n = 1 << log_n
    rev = np.array([int(format(i, f"0{log_n}b")[::-1], 2) for i in range(n)])
    for region in (1, 2):
        primes = ctx.level_primes(q, -region)
        for j in sorted({0, len(primes) // 2, len(primes) - 1}):
            p = int(primes[j])
            psi = mm.root_2n(p, n)
            for tab, base in zip(ctx.level_twiddles32(q, region, j), (psi, pow(psi, p - 2, p))):
                w = np.ones(n, np.uint64)
                for i in range(1, n):
                    w[i] = w[i - 1] * base % p
                want_w = np.zeros(n, np.uint64)
                want_w[rev] = w
                want_q = (want_w << np.uint64(32)) // np.uint64(p)
                assert np.array_equal(tab[:, 0].astype(np.uint64), want_w), (region, j)
                assert np.array_equal(tab[:, 1].astype(np.uint64), want_q), (region, j)
    ctx.close()
