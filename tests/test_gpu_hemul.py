"""HE Mul (+ relinearize + rescale) on the GPU, bit-exact against the
reference: golden fixtures, golden digests of the seed-7 bench protocol
(bench.cpp:49-124) and the oracles. Restates test_heaan.cpp:129-199 and
test_cli.cpp:141-170 (digest identity)."""
from __future__ import annotations

import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import random_poly

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


# he_mul engines: prime basis (HEMUL_OPT_BASIS) x base-conversion engine
# (HEMUL_OPT_TENSOR_CORES, 30-bit basis only); results must not depend on them
BASES = ["32tc", "32imad", "64"]
# + the tensor-core engine with natural-order pass-A rows (HEMUL_OPT_TRANSPOSED
# off; the default lays them out column-major at log N >= 15)
BASES_PAPER = BASES + ["32tc-natural"]


def _word(basis) -> int:
    return int(str(basis)[:2])


def _ctx(cfg, basis="32tc"):
    from paper_2003_04510_b200.hemul import Context, make_params

    ctx = Context(make_params(*cfg))
    ctx.set_basis(_word(basis))
    ctx.set_tensor_cores("tc" in str(basis))
    ctx.set_transposed(not str(basis).endswith("natural"))
    return ctx


def _digest(log_q, ax, bx):
    from paper_2003_04510_b200.hemul import ciphertext_digest

    return ciphertext_digest(log_q, ax, bx)


def test_s_bench_golden_fixture():
    g = np.load(GOLDEN / "s_bench.npz")
    digests = json.loads((GOLDEN / "digests.json").read_text())
    ctx = _ctx((30, 4, 13))
    q = int(g["log_q"])
    oa, ob = ctx.he_mul((g["c1ax"], g["c1bx"]), (g["c2ax"], g["c2bx"]), q,
                        evk=(g["evkax"], g["evkbx"]))
    assert np.array_equal(oa, g["outax"])
    assert np.array_equal(ob, g["outbx"])
    assert f"{_digest(q - 30, oa, ob):016x}" == digests["S"]["digest"]


def test_small_random_two_levels_golden():
    g = np.load(GOLDEN / "small_random.npz")
    cfg = tuple(int(v) for v in g["params"])
    ctx = _ctx(cfg)
    evk = (g["evkax"], g["evkbx"])
    for lvl in (0, 1):
        q = int(g[f"log_q_{lvl}"])
        oa, ob = ctx.he_mul((g[f"c1ax_{lvl}"], g[f"c1bx_{lvl}"]),
                            (g[f"c2ax_{lvl}"], g[f"c2bx_{lvl}"]), q, evk=evk)
        assert np.array_equal(oa, g[f"outax_{lvl}"])
        assert np.array_equal(ob, g[f"outbx_{lvl}"])


@pytest.mark.parametrize("basis", BASES)
@pytest.mark.parametrize("cfg", [(30, 4, 13), (30, 6, 11), (30, 10, 13), (20, 4, 10)])
def test_random_inputs_every_level_vs_oracle(cfg, basis, restated):
    """Random residues at every level of the ladder (the level LRU evicts,
    heaan.cpp:119-150) against the C restatement."""
    ctx = _ctx(cfg, basis)
    assert ctx.mul_basis(ctx.params.log_q_max)[0] == _word(basis)
    p = ctx.params
    rng = np.random.default_rng(sum(cfg))
    evk = (random_poly(rng, p.n, 2 * p.log_q_max), random_poly(rng, p.n, 2 * p.log_q_max))
    for log_q in range(p.log_q_max, 2 * p.log_p - 1, -p.log_p):
        c1 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        c2 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, p.log_q_max, log_q, c1, c2, evk)
        assert st == 0
        oa, ob = ctx.he_mul(c1, c2, log_q, evk=evk)
        assert np.array_equal(oa, wa), log_q
        assert np.array_equal(ob, wb), log_q


@pytest.mark.parametrize("basis", BASES)
@pytest.mark.parametrize("cfg", [(30, 4, 13), (30, 10, 12), (30, 6, 11)])
def test_exact_fixup_path_matches(cfg, basis, restated):
    """The finisher's exact big-integer fix-up (normally taken with
    probability 2^-64 per coefficient) forced on every coefficient."""
    ctx = _ctx(cfg, basis)
    ctx.set_force_exact(True)
    p = ctx.params
    rng = np.random.default_rng(77)
    evk = (random_poly(rng, p.n, 2 * p.log_q_max), random_poly(rng, p.n, 2 * p.log_q_max))
    for log_q in (p.log_q_max, 2 * p.log_p):
        c1 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        c2 = (random_poly(rng, p.n, log_q), random_poly(rng, p.n, log_q))
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, p.log_q_max, log_q, c1, c2, evk)
        oa, ob = ctx.he_mul(c1, c2, log_q, evk=evk)
        assert np.array_equal(oa, wa) and np.array_equal(ob, wb), log_q


@pytest.mark.parametrize("basis", BASES)
def test_edge_inputs_zero_and_all_ones(basis, restated):
    cfg = (30, 4, 10)
    ctx = _ctx(cfg, basis)
    p = ctx.params
    q = p.log_q_max
    rng = np.random.default_rng(1)
    evk = (random_poly(rng, p.n, 2 * q), random_poly(rng, p.n, 2 * q))
    ones = np.full((p.n, 2), np.uint64(0xFFFFFFFFFFFFFFFF))
    ones[:, -1] &= np.uint64((1 << (q % 64)) - 1)
    zero = np.zeros_like(ones)
    for c1, c2 in [((zero, zero), (zero, zero)), ((ones, ones), (ones, ones)),
                   ((ones, zero), (zero, ones))]:
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, q, q, c1, c2, evk)
        oa, ob = ctx.he_mul(c1, c2, q, evk=evk)
        assert np.array_equal(oa, wa) and np.array_equal(ob, wb)


@pytest.mark.parametrize("basis", BASES)
def test_batch_equals_singles(basis, restated):
    cfg = (30, 4, 12)
    ctx = _ctx(cfg, basis)
    p = ctx.params
    q = p.log_q_max
    rng = np.random.default_rng(9)
    evk = (random_poly(rng, p.n, 2 * q), random_poly(rng, p.n, 2 * q))
    B = 3
    c1 = [np.stack([random_poly(rng, p.n, q) for _ in range(B)]) for _ in range(2)]
    c2 = [np.stack([random_poly(rng, p.n, q) for _ in range(B)]) for _ in range(2)]
    oa, ob = ctx.he_mul((c1[0], c1[1]), (c2[0], c2[1]), q, evk=evk)
    assert oa.shape == (B, p.n, 2)
    for b in range(B):
        sa, sb = ctx.he_mul((c1[0][b], c1[1][b]), (c2[0][b], c2[1][b]), q, evk=evk)
        assert np.array_equal(oa[b], sa) and np.array_equal(ob[b], sb)
    st, wa, wb = restated.he_mul(p.log_n, p.log_p, q, q, (c1[0][1], c1[1][1]),
                                 (c2[0][1], c2[1][1]), evk)
    assert np.array_equal(oa[1], wa) and np.array_equal(ob[1], wb)


def test_errors_match_reference_kinds():
    """heaan.cpp:341-345: mismatch -> invalid_argument, depth -> runtime_error
    (test_heaan.cpp:169-182)."""
    ctx = _ctx((30, 4, 10))
    p = ctx.params
    z = np.zeros((p.n, 2), np.uint64)
    with pytest.raises(ValueError, match="ciphertext modulus mismatch"):
        ctx.he_mul((z, z), (z, z), 120, c2_log_q=90, evk=(np.zeros((p.n, 4), np.uint64),) * 2)
    z1 = np.zeros((p.n, 1), np.uint64)
    with pytest.raises(RuntimeError, match="multiplicative depth exhausted"):
        ctx.he_mul((z1, z1), (z1, z1), 30, evk=(np.zeros((p.n, 4), np.uint64),) * 2)
    with pytest.raises(RuntimeError, match="modulus exhausted; cannot rescale"):
        ctx.rescale((z1, z1), 30)


def test_rescale_matches_reference(reference):
    cfg = (30, 4, 10)
    ctx = _ctx(cfg)
    p = ctx.params
    rng = np.random.default_rng(4)
    a = random_poly(rng, p.n, 120)
    b = random_poly(rng, p.n, 120)
    oa, ob = ctx.rescale((a, b), 120)
    assert np.array_equal(oa, reference.shift_right(p.n, 120, 30, a))
    assert np.array_equal(ob, reference.shift_right(p.n, 120, 30, b))


def test_device_resident_inputs_torch():
    torch = pytest.importorskip("torch")
    g = np.load(GOLDEN / "s_bench.npz")
    ctx = _ctx((30, 4, 13))
    q = int(g["log_q"])
    dev = {k: torch.from_numpy(g[k]).cuda() for k in ("c1ax", "c1bx", "c2ax", "c2bx",
                                                       "evkax", "evkbx")}
    launches0 = ctx.launch_count()
    oa, ob = ctx.he_mul((dev["c1ax"], dev["c1bx"]), (dev["c2ax"], dev["c2bx"]), q,
                        evk=(dev["evkax"], dev["evkbx"]))
    ctx.synchronize()
    assert oa.is_cuda
    assert np.array_equal(oa.cpu().numpy(), g["outax"])
    assert np.array_equal(ob.cpu().numpy(), g["outbx"])
    assert ctx.launch_count() > launches0


def test_stage_timing_buckets():
    g = np.load(GOLDEN / "s_bench.npz")
    ctx = _ctx((30, 4, 13))
    ctx.enable_stage_timing(True)
    q = int(g["log_q"])
    ctx.he_mul((g["c1ax"], g["c1bx"]), (g["c2ax"], g["c2bx"]), q, evk=(g["evkax"], g["evkbx"]))
    ms = ctx.stage_ms()
    assert set(ms) == {"crt", "ntt", "intt", "icrt", "extra"}
    assert all(v > 0 for v in ms.values())


def test_basis_switch_and_counts():
    """The 30-bit basis covers every ring degree the parameter table allows;
    switching bases re-derives the evk forms and gives the same ciphertext."""
    g = np.load(GOLDEN / "s_bench.npz")
    ctx = _ctx((30, 4, 13), 32)
    q = int(g["log_q"])
    word, np1, np2 = ctx.mul_basis(q)
    assert word == 32 and np2 > len(ctx.level_primes(q, 2))
    assert int(ctx.level_primes(q, -1).max()) < (1 << 30)
    evk = (g["evkax"], g["evkbx"])
    outs = []
    for basis in (32, 64, 32):
        ctx.set_basis(basis)
        outs.append(ctx.he_mul((g["c1ax"], g["c1bx"]), (g["c2ax"], g["c2bx"]), q, evk=evk))
    for oa, ob in outs:
        assert np.array_equal(oa, g["outax"]) and np.array_equal(ob, g["outbx"])


def test_region2_shrinks_with_level():
    """The 30-bit basis takes the evk mod 2^(log_q + log_Q) before its CRT
    (context.cu evk_forms), so region 2 covers |d2 evk| < n q^2 Q plus the
    iCRT headroom and shrinks with the level; the w64 basis keeps the
    reference's rule (log_q + 2 log_Q + log_n, heaan.cpp:139-143)."""
    ctx = _ctx((30, 4, 13), 32)
    log_qm, log_n = ctx.params.log_q_max, ctx.params.log_n
    prev = None
    for q in (log_qm, log_qm - 30, log_qm - 60):
        p2 = [int(x) for x in ctx.level_primes(q, -2)]
        bits = math.prod(p2).bit_length()
        vbits = 2 * q + log_qm + log_n
        assert bits - 2 - vbits >= 4                              # iCRT headroom
        assert math.prod(p2[:-1]).bit_length() - 2 - vbits < 4   # and no more primes
        if prev is not None:
            assert len(p2) < prev
        prev = len(p2)
    ctx.set_basis(64)
    q = log_qm - 60
    p2 = [int(x) for x in ctx.level_primes(q, -2)]
    assert math.prod(p2).bit_length() > q + 2 * log_qm + log_n


@pytest.mark.slow
@pytest.mark.parametrize("basis", BASES_PAPER)
@pytest.mark.parametrize("name", ["logN14_logQ300", "logN15_logQ600", "M", "X"])
def test_bench_protocol_digest_paper_scale(name, basis, reference):
    """Digest of he_mul on the reference's own seed-7 keys and ciphertexts
    equals the reference's."""
    d = json.loads((GOLDEN / "digests.json").read_text())[name]
    cfg = tuple(d["params"])
    inp = reference.bench_inputs(*cfg, seed=7)
    ctx = _ctx(cfg, basis)
    q = inp["log_q_max"]
    oa, ob = ctx.he_mul(inp["c1"], inp["c2"], q, evk=inp["evk"])
    assert f"{_digest(q - cfg[0], oa, ob):016x}" == d["digest"]


# ---- paper-scale parity below the fresh modulus ------------------------------
# Levels of the M and X ladders (heaan.cpp:339-410 at log_q < log_Q): the
# region tables, the split point and the iCRT / finisher byte windows all
# change with log_q. Random ciphertexts (SURVEY §8(d) throughput inputs) and
# one random evk per config; the reference's own he_mul (oracle/_ref, all host
# threads) computes each expected output once, shared by the three engines.
PAPER_LADDERS = {"X": ((30, 80, 0), [2400, 1800, 1200, 60]),
                 "M": ((30, 40, 0), [1200, 630, 60])}
_REF_CACHE: dict = {}


def _paper_case(name, log_q, reference):
    key = (name, log_q)
    if key not in _REF_CACHE:
        import os

        cfg, _ = PAPER_LADDERS[name]
        log_n, n, qmax = reference.make_params(*cfg)
        rng = np.random.default_rng(1000 + log_q)
        if (name, "evk") not in _REF_CACHE:
            erng = np.random.default_rng(7)
            _REF_CACHE[(name, "evk")] = (random_poly(erng, n, 2 * qmax),
                                         random_poly(erng, n, 2 * qmax))
        evk = _REF_CACHE[(name, "evk")]
        c1 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        c2 = (random_poly(rng, n, log_q), random_poly(rng, n, log_q))
        st, wa, wb = reference.he_mul(*cfg, log_q, c1, c2, evk, threads=os.cpu_count() or 1)
        assert st == 0, reference.err()
        _REF_CACHE[key] = (c1, c2, evk, wa, wb)
    return _REF_CACHE[key]


@pytest.mark.slow
@pytest.mark.parametrize("basis", BASES)
@pytest.mark.parametrize("name", ["M", "X"])
def test_paper_scale_ladder_levels_vs_reference(name, basis, reference):
    cfg, levels = PAPER_LADDERS[name]
    ctx = _ctx(cfg, basis)
    for log_q in levels:
        c1, c2, evk, wa, wb = _paper_case(name, log_q, reference)
        oa, ob = ctx.he_mul(c1, c2, log_q, evk=evk)
        assert np.array_equal(oa, wa), (name, log_q, basis)
        assert np.array_equal(ob, wb), (name, log_q, basis)
    ctx.close()


# ---- evk identity and batch limits --------------------------------

def test_two_evks_at_one_level_in_one_context(restated):
    """The cached evk forms are keyed by the key's identity (heaan.cpp:152):
    a different evk at an already-warm level must not reuse the old forms."""
    cfg = (30, 4, 10)
    ctx = _ctx(cfg)
    p = ctx.params
    q = p.log_q_max
    rng = np.random.default_rng(31)
    evks = [(random_poly(rng, p.n, 2 * q), random_poly(rng, p.n, 2 * q)) for _ in range(2)]
    c1 = (random_poly(rng, p.n, q), random_poly(rng, p.n, q))
    c2 = (random_poly(rng, p.n, q), random_poly(rng, p.n, q))
    for evk in (evks[0], evks[1], evks[0], evks[1]):
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, q, q, c1, c2, evk)
        oa, ob = ctx.he_mul(c1, c2, q, evk=evk)
        assert np.array_equal(oa, wa) and np.array_equal(ob, wb)
    # an equal-content copy is a different key object: rebuilt, same result
    copy = (evks[1][0].copy(), evks[1][1].copy())
    oa2, ob2 = ctx.he_mul(c1, c2, q, evk=copy)
    assert np.array_equal(oa2, oa) and np.array_equal(ob2, ob)


@pytest.mark.parametrize("device", [False, True], ids=["host", "device"])
def test_batch_beyond_grid_row_limit(device):
    """More rows than gridDim.y allows (65535) in one launch: the context runs
    the batch in sub-batches (context.cu row limits)."""
    torch = pytest.importorskip("torch")
    cfg = (30, 4, 10)
    ctx = _ctx(cfg)
    p = ctx.params
    q = p.log_q_max
    info = ctx.engine_info(q)
    rows_per_pair = max(8 * info["np1"], 2 * info["np2"])
    B = 65535 // rows_per_pair + 37
    rng = np.random.default_rng(5)
    evk = (random_poly(rng, p.n, 2 * q), random_poly(rng, p.n, 2 * q))
    base = [[random_poly(rng, p.n, q) for _ in range(4)] for _ in range(3)]
    singles = [ctx.he_mul((b[0], b[1]), (b[2], b[3]), q, evk=evk) for b in base]
    polys = [np.stack([base[i % 3][t] for i in range(B)]) for t in range(4)]
    if device:
        polys = [torch.from_numpy(x).cuda() for x in polys]
    oa, ob = ctx.he_mul((polys[0], polys[1]), (polys[2], polys[3]), q, evk=evk)
    if device:
        ctx.synchronize()
        oa, ob = oa.cpu().numpy(), ob.cpu().numpy()
    assert oa.shape[0] == B
    for i in (0, 1, 2, B // 2, B - 1):
        assert np.array_equal(oa[i], singles[i % 3][0]) and np.array_equal(ob[i], singles[i % 3][1])


# ---- device-resident chains -----------------------------

def _mod_down_np(a, log_q, new_log_q):
    """poly_mod_down (poly.cpp:117-127) on a host BigPoly."""
    L = (new_log_q + 63) // 64
    out = np.ascontiguousarray(a[..., :L]).copy()
    if new_log_q % 64:
        out[..., -1] &= np.uint64((1 << (new_log_q % 64)) - 1)
    return out


@pytest.mark.slow
@pytest.mark.parametrize("basis", ["32tc", "64"])
def test_device_chain_paper_scale_vs_reference(basis, reference):
    """A 4-step HE Mul chain at N=2^17 / logQ=2400 with every operand resident
    in HBM (upload once, mod_down on the device, download once) equals the
    reference's he_mul applied step by step."""
    import os

    cfg = (30, 80, 0)
    key = ("chain", cfg)
    if key not in _REF_CACHE:
        log_n, n, qmax = reference.make_params(*cfg)
        rng = np.random.default_rng(4242)
        evk = (random_poly(rng, n, 2 * qmax), random_poly(rng, n, 2 * qmax))
        acc = (random_poly(rng, n, qmax), random_poly(rng, n, qmax))
        fresh = [(random_poly(rng, n, qmax), random_poly(rng, n, qmax)) for _ in range(4)]
        want, q = [], qmax
        cur = acc
        for c in fresh:
            cd = (_mod_down_np(c[0], qmax, q), _mod_down_np(c[1], qmax, q))
            st, wa, wb = reference.he_mul(*cfg, q, cur, cd, evk, threads=os.cpu_count() or 1)
            assert st == 0, reference.err()
            cur = (wa, wb)
            q -= cfg[0]
            want.append(cur)
        _REF_CACHE[key] = (evk, acc, fresh, want)
    evk, acc, fresh, want = _REF_CACHE[key]
    ctx = _ctx(cfg, basis)
    ctx.set_level_cache(4)
    qmax = ctx.params.log_q_max
    dacc = ctx.upload(acc, qmax)
    dfresh = [ctx.upload(c, qmax) for c in fresh]
    outs = []
    for k, dc in enumerate(dfresh):
        if dc.log_q > dacc.log_q:
            dc = ctx.mod_down_dev(dc, dacc.log_q)
        dacc = ctx.he_mul_dev(dacc, dc, evk=evk)
        outs.append(dacc)
    for k, (o, w) in enumerate(zip(outs, want)):
        ga, gb = o.download()
        assert o.log_q == qmax - (k + 1) * 30
        assert np.array_equal(ga, w[0]) and np.array_equal(gb, w[1]), k


def test_device_handles_small_chain(restated):
    """Handles: upload / he_mul_dev / rescale_dev / mod_down_dev / download
    against the C restatement and the host-buffer path."""
    cfg = (30, 6, 11)
    ctx = _ctx(cfg)
    p = ctx.params
    q = p.log_q_max
    rng = np.random.default_rng(11)
    evk = (random_poly(rng, p.n, 2 * q), random_poly(rng, p.n, 2 * q))
    c1 = (random_poly(rng, p.n, q), random_poly(rng, p.n, q))
    c2 = (random_poly(rng, p.n, q), random_poly(rng, p.n, q))
    d1, d2 = ctx.upload(c1, q), ctx.upload(c2, q, asynchronous=True)
    assert np.array_equal(d1.download()[0], c1[0])
    r = ctx.he_mul_dev(d1, d2, evk=evk)
    st, wa, wb = restated.he_mul(p.log_n, p.log_p, q, q, c1, c2, evk)
    ga, gb = r.download()
    assert r.log_q == q - 30 and np.array_equal(ga, wa) and np.array_equal(gb, wb)
    rs = ctx.rescale_dev(r)
    ha, hb = ctx.rescale((wa, wb), q - 30)
    sa, sb = rs.download()
    assert np.array_equal(sa, ha) and np.array_equal(sb, hb)
    md = ctx.mod_down_dev(d1, q - 61)
    ma, mb = md.download()
    assert np.array_equal(ma, _mod_down_np(c1[0], q, q - 61))
    assert np.array_equal(mb, _mod_down_np(c1[1], q, q - 61))
    with pytest.raises(ValueError, match="ciphertext modulus mismatch"):
        ctx.he_mul_dev(r, d1, evk=evk)
    # batched handles
    B = 3
    cb1 = [np.stack([random_poly(rng, p.n, q) for _ in range(B)]) for _ in range(2)]
    cb2 = [np.stack([random_poly(rng, p.n, q) for _ in range(B)]) for _ in range(2)]
    rb = ctx.he_mul_dev(ctx.upload(tuple(cb1), q), ctx.upload(tuple(cb2), q), evk=evk)
    ba, bb = rb.download()
    ha, hb = ctx.he_mul(tuple(cb1), tuple(cb2), q, evk=evk)
    assert np.array_equal(ba, ha) and np.array_equal(bb, hb)


def test_torch_tensors_follow_torch_stream(restated):
    """A Context without an explicit stream runs calls on torch CUDA tensors
    on torch's current stream (the default stream maps to cudaStreamLegacy):
    inputs produced by torch kernels just before the call and outputs read by
    torch right after are ordered without a host sync."""
    import torch

    cfg = (30, 4, 13)
    ctx = _ctx(cfg)
    p = ctx.params
    q = p.log_q_max
    for seed in range(3):
        g = torch.Generator(device="cuda")
        g.manual_seed(seed)

        def rnd(bits):
            t = torch.randint(-(2**63), 2**63 - 1, (p.n, (bits + 63) // 64), generator=g,
                              device="cuda", dtype=torch.int64)
            if bits % 64:
                t[:, -1] &= (1 << (bits % 64)) - 1
            return t.view(torch.uint64)

        c1, c2, evk = (rnd(q), rnd(q)), (rnd(q), rnd(q)), (rnd(2 * q), rnd(2 * q))
        oa, ob = ctx.he_mul(c1, c2, q, evk=evk, evk_id=0)  # no synchronize in between
        ga, gb = oa.cpu().numpy(), ob.cpu().numpy()
        h = lambda t: t.cpu().numpy()  # noqa: E731
        st, wa, wb = restated.he_mul(p.log_n, p.log_p, q, q, (h(c1[0]), h(c1[1])),
                                     (h(c2[0]), h(c2[1])), (h(evk[0]), h(evk[1])))
        assert st == 0 and np.array_equal(ga, wa) and np.array_equal(gb, wb), seed
    ctx.close()
