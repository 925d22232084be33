"""ctypes bindings of the TEST-ONLY oracles (never imported by the product).

* ``Restated`` — oracle/liboracle.so, the C restatement (oracle/hemul_oracle.h)
* ``Reference`` — oracle/_ref/libhemul_ref.so, the reference itself compiled
  from /root/reference/proj/core by oracle/Makefile (oracle/ref_shim.cpp)
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
RESTATED_SO = ROOT / "oracle" / "liboracle.so"
REFERENCE_SO = ROOT / "oracle" / "_ref" / "libhemul_ref.so"

_p = ctypes.c_void_p
_i = ctypes.c_int
_u64 = ctypes.c_uint64


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.uint64 and a.flags["C_CONTIGUOUS"], a.dtype
    return a.ctypes.data


def limbs(bits: int) -> int:
    return (bits + 63) // 64


class Restated:
    def __init__(self, path: Path = RESTATED_SO):
        self.lib = ctypes.CDLL(str(path))
        L = self.lib
        L.orc_region_primes.argtypes = [_i, _i, _i, _i, _p, _p, _i]
        L.orc_region_primes.restype = _i
        L.orc_ntt_tables.argtypes = [_u64, _u64, _i, _p, _p, _p]
        L.orc_ntt_forward.argtypes = [_p, _i, _u64, _p]
        L.orc_ntt_inverse.argtypes = [_p, _i, _u64, _p, _u64]
        L.orc_crt.argtypes = [_p, _i, _i, _p, _i, _p]
        L.orc_pointwise.argtypes = [_p, _p, _i, _p, _i, _p]
        L.orc_icrt.argtypes = [_p, _i, _p, _i, _i, _p]
        L.orc_shift_right.argtypes = [_p, _i, _i, _i, _p]
        L.orc_he_mul.argtypes = [_i, _i, _i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p]
        L.orc_he_mul.restype = _i
        L.orc_digest.argtypes = [_i, _i, _p, _p]
        L.orc_digest.restype = _u64

    def region_primes(self, region, log_q, log_q_max, log_n):
        np_ = self.lib.orc_region_primes(region, log_q, log_q_max, log_n, None, None, 0)
        pr = np.zeros(np_, np.uint64)
        rt = np.zeros(np_, np.uint64)
        self.lib.orc_region_primes(region, log_q, log_q_max, log_n, _ptr(pr), _ptr(rt), np_)
        return pr, rt

    def ntt_tables(self, p, psi, log_n):
        n = 1 << log_n
        tw = np.zeros(n, np.uint64)
        itw = np.zeros(n, np.uint64)
        ninv = np.zeros(1, np.uint64)
        self.lib.orc_ntt_tables(int(p), int(psi), log_n, _ptr(tw), _ptr(itw), _ptr(ninv))
        return tw, itw, int(ninv[0])

    def ntt(self, rows, primes, roots, log_n, inverse=False):
        """Row r transformed mod primes[r % np] (in a copy)."""
        out = np.array(rows, dtype=np.uint64, copy=True).reshape(-1, 1 << log_n)
        tabs = [self.ntt_tables(p, r, log_n) for p, r in zip(primes, roots)]
        for r in range(out.shape[0]):
            j = r % len(primes)
            row = np.ascontiguousarray(out[r])
            tw, itw, ninv = tabs[j]
            if inverse:
                self.lib.orc_ntt_inverse(_ptr(row), log_n, int(primes[j]), _ptr(itw), ninv)
            else:
                self.lib.orc_ntt_forward(_ptr(row), log_n, int(primes[j]), _ptr(tw))
            out[r] = row
        return out

    def crt(self, poly, n, limbs_, primes):
        out = np.zeros((len(primes), n), np.uint64)
        self.lib.orc_crt(_ptr(np.ascontiguousarray(poly)), n, limbs_, _ptr(primes), len(primes),
                         _ptr(out))
        return out

    def pointwise(self, a, b, primes, n):
        out = np.zeros_like(a)
        self.lib.orc_pointwise(_ptr(a), _ptr(b), n, _ptr(primes), len(primes), _ptr(out))
        return out

    def icrt(self, rns, n, primes, target_bits):
        out = np.zeros((n, limbs(target_bits)), np.uint64)
        self.lib.orc_icrt(_ptr(np.ascontiguousarray(rns)), n, _ptr(primes), len(primes),
                          target_bits, _ptr(out))
        return out

    def shift_right(self, a, n, log_q, bits):
        out = np.zeros((n, limbs(log_q - bits)), np.uint64)
        self.lib.orc_shift_right(_ptr(a), n, log_q, bits, _ptr(out))
        return out

    def he_mul(self, log_n, log_p, log_q_max, log_q, c1, c2, evk, c2_log_q=None):
        n = 1 << log_n
        lo = limbs(log_q - log_p)
        oa = np.zeros((n, lo), np.uint64)
        ob = np.zeros((n, lo), np.uint64)
        st = self.lib.orc_he_mul(log_n, log_p, log_q_max, log_q,
                                 log_q if c2_log_q is None else c2_log_q,
                                 _ptr(c1[0]), _ptr(c1[1]), _ptr(c2[0]), _ptr(c2[1]),
                                 _ptr(evk[0]), _ptr(evk[1]), _ptr(oa), _ptr(ob))
        return st, oa, ob

    def digest(self, log_q, n, ax, bx):
        return int(self.lib.orc_digest(log_q, n, _ptr(ax), _ptr(bx)))


class Reference:
    def __init__(self, path: Path = REFERENCE_SO):
        self.lib = ctypes.CDLL(str(path))
        L = self.lib
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_make_params.argtypes = [_i, _i, _i, _p]
        L.ref_level_primes.argtypes = [_i, _i, _i, _i, _p, _p, _i]
        L.ref_bench_inputs.argtypes = [_i, _i, _i, _u64, _p, _p, _p, _p, _p, _p, _p]
        L.ref_he_mul.argtypes = [_i, _i, _i, _i, _p, _p, _p, _p, _i, _p, _p, _p, _p, _i, _i]
        L.ref_run_bench.argtypes = [_i, _i, _i, _u64, _i, _i, _i, _p, _p]
        L.ref_digest.argtypes = [_i, _i, _p, _p]
        L.ref_digest.restype = _u64
        L.ref_prepare.argtypes = [_i, _i, _i, _i, _i, _p, _p, _i]
        L.ref_ntt.argtypes = [_i, _i, _i, _i, _p, _i]
        L.ref_finish.argtypes = [_i, _i, _i, _i, _p, _p, _i]
        L.ref_pointwise.argtypes = [_i, _i, _i, _i, _p, _p, _p]
        L.ref_shift_right.argtypes = [_i, _i, _i, _p, _p]
        L.ref_time_he_mul.argtypes = [_i, _i, _i, _u64, _i, _i, _i, _p, _p]
        L.ref_time_ntt.argtypes = [_i, _i, _i, _i, _i, _i, _p]
        L.ref_counters.argtypes = [_i, _i, _i, _u64, _i, _i, _p]

    def counters(self, log_p, depth, log_n_override, seed=7, four_products=False,
                 periodic=False):
        """Scheme::counters after one he_mul: 5 stages x {mul, adc, modmul, addsub}."""
        out = np.zeros(20, np.uint64)
        st = self.lib.ref_counters(log_p, depth, log_n_override, seed, int(four_products),
                                   int(periodic), _ptr(out))
        assert st == 0, self.err()
        return [int(v) for v in out]

    def err(self):
        return self.lib.ref_last_error().decode()

    def make_params(self, log_p, depth, log_n_override=0):
        out = np.zeros(3, np.int32)
        assert self.lib.ref_make_params(log_p, depth, log_n_override, out.ctypes.data) == 0
        return int(out[0]), int(out[1]), int(out[2])

    def level_primes(self, region, log_q, log_q_max, log_n):
        cap = 512
        pr = np.zeros(cap, np.uint64)
        rt = np.zeros(cap, np.uint64)
        np_ = self.lib.ref_level_primes(region, log_q, log_q_max, log_n, _ptr(pr), _ptr(rt), cap)
        assert np_ > 0, self.err()
        return pr[:np_].copy(), rt[:np_].copy()

    def bench_inputs(self, log_p, depth, log_n_override=0, seed=7):
        log_n, n, log_q_max = self.make_params(log_p, depth, log_n_override)
        L, Le = limbs(log_q_max), limbs(2 * log_q_max)
        c = [np.zeros((n, L), np.uint64) for _ in range(4)]
        e = [np.zeros((n, Le), np.uint64) for _ in range(2)]
        sk = np.zeros(n, np.int32)
        st = self.lib.ref_bench_inputs(log_p, depth, log_n_override, seed, *map(_ptr, c),
                                       *map(_ptr, e), sk.ctypes.data)
        assert st == 0, self.err()
        return {"c1": (c[0], c[1]), "c2": (c[2], c[3]), "evk": (e[0], e[1]), "sk": sk,
                "log_n": log_n, "n": n, "log_q_max": log_q_max}

    def he_mul(self, log_p, depth, log_n_override, log_q, c1, c2, evk, c2_log_q=None,
               threads=1, radix_log=1):
        log_n, n, _ = self.make_params(log_p, depth, log_n_override)
        lo = limbs(log_q - log_p)
        oa = np.zeros((n, lo), np.uint64)
        ob = np.zeros((n, lo), np.uint64)
        st = self.lib.ref_he_mul(log_p, depth, log_n_override, log_q, _ptr(c1[0]), _ptr(c1[1]),
                                 _ptr(c2[0]), _ptr(c2[1]), log_q if c2_log_q is None else c2_log_q,
                                 _ptr(evk[0]), _ptr(evk[1]), _ptr(oa), _ptr(ob), threads,
                                 radix_log)
        return st, oa, ob

    def run_bench(self, log_p, depth, log_n_override=0, seed=7, reps=1, threads=1, radix_log=1):
        ms = np.zeros(7, np.float64)
        dig = np.zeros(1, np.uint64)
        st = self.lib.ref_run_bench(log_p, depth, log_n_override, seed, reps, threads, radix_log,
                                    ms.ctypes.data, dig.ctypes.data)
        assert st == 0, self.err()
        keys = ("crt", "ntt", "intt", "icrt", "extra", "total_mean", "total_median")
        return int(dig[0]), dict(zip(keys, ms.tolist()))

    def digest(self, log_q, n, ax, bx):
        return int(self.lib.ref_digest(log_q, n, _ptr(ax), _ptr(bx)))

    def time_ntt(self, log_n, np_, threads=1, radix_log=4, reps=1, inverse=False):
        """Wall ms of `reps` reference ntt_forward / ntt_inverse calls over np_
        rows of 2^log_n (bench_ntt.cpp protocol)."""
        ms = np.zeros(reps, np.float64)
        st = self.lib.ref_time_ntt(log_n, np_, threads, radix_log, reps, int(inverse),
                                   ms.ctypes.data)
        assert st == 0, self.err()
        return ms.tolist()

    def time_he_mul(self, log_p, depth, log_n_override=0, seed=1, reps=1, threads=1,
                    radix_log=1):
        """Wall ms of `reps` warm he_mul calls on random inputs (+ digest)."""
        ms = np.zeros(reps, np.float64)
        dig = np.zeros(1, np.uint64)
        st = self.lib.ref_time_he_mul(log_p, depth, log_n_override, seed, reps, threads,
                                      radix_log, ms.ctypes.data, dig.ctypes.data)
        assert st == 0, self.err()
        return ms.tolist(), int(dig[0])

    def prepare(self, region, log_q, log_q_max, log_n, in_bits, poly, np_, stop_after_crt=False):
        out = np.zeros((np_, 1 << log_n), np.uint64)
        st = self.lib.ref_prepare(region, log_q, log_q_max, log_n, in_bits,
                                  _ptr(np.ascontiguousarray(poly)), _ptr(out), int(stop_after_crt))
        assert st == 0, self.err()
        return out

    def ntt(self, region, log_q, log_q_max, log_n, data, inverse=False):
        d = np.array(data, dtype=np.uint64, copy=True)
        assert self.lib.ref_ntt(region, log_q, log_q_max, log_n, _ptr(d), int(inverse)) == 0
        return d

    def finish(self, region, log_q, log_q_max, log_n, rns, target_bits, skip_intt=False):
        out = np.zeros((1 << log_n, limbs(target_bits)), np.uint64)
        st = self.lib.ref_finish(region, log_q, log_q_max, log_n, _ptr(np.ascontiguousarray(rns)),
                                 _ptr(out), int(skip_intt))
        assert st == 0, self.err()
        return out

    def pointwise(self, region, log_q, log_q_max, log_n, a, b):
        out = np.zeros_like(a)
        assert self.lib.ref_pointwise(region, log_q, log_q_max, log_n, _ptr(a), _ptr(b),
                                      _ptr(out)) == 0
        return out

    def shift_right(self, n, log_q, bits, a):
        out = np.zeros((n, limbs(log_q - bits)), np.uint64)
        assert self.lib.ref_shift_right(n, log_q, bits, _ptr(a), _ptr(out)) == 0
        return out


def random_poly(rng: np.random.Generator, n: int, bits: int) -> np.ndarray:
    """Uniform coefficients in [0, 2^bits) in BigPoly layout (top limb masked,
    poly.cpp:38-44)."""
    L = limbs(bits)
    a = rng.integers(0, 2**64, size=(n, L), dtype=np.uint64, endpoint=False)
    if bits % 64:
        a[:, -1] &= np.uint64((1 << (bits % 64)) - 1)
    return a
