"""Test-side residue arithmetic for the stage-by-stage parity tests of the
30-bit basis (tests/test_gpu_basis32.py). Test infrastructure only.

Everything here restates the reference's polynomial-product algebra
(polymul.cpp:7-43: CRT -> negacyclic product per prime -> centred iCRT) with
arbitrary primes p < 2^31, vectorised over rows with numpy:

* ``residues``      crt_forward (rns.cpp:43-106): v mod p_j from the BigPoly limbs
* ``negacyclic``    iNTT(NTT(a) . NTT(b)) (ntt.cpp:59-137 + rns.cpp:108-130) —
                    root-independent, so any primitive 2n-th root gives the
                    reference's coefficients
* ``centred_lift``  icrt (rns.cpp:132-190): the integer in (-P/2, P/2]

The helpers are pinned against the C restatement (oracle/hemul_oracle.c) by
tests/test_modmath.py.
"""
from __future__ import annotations

import numpy as np


def poly_ints(a: np.ndarray) -> list[int]:
    """BigPoly (n, limbs) u64 -> Python ints (little-endian limbs, poly.hpp:15-26)."""
    a = np.ascontiguousarray(a, dtype=np.uint64)
    raw = a.tobytes()
    w = a.shape[1] * 8
    return [int.from_bytes(raw[i * w:(i + 1) * w], "little") for i in range(a.shape[0])]


def ints_poly(vals: list[int], bits: int) -> np.ndarray:
    """Python ints (taken mod 2^bits) -> BigPoly (n, ceil(bits/64)) u64."""
    L = (bits + 63) // 64
    mask = (1 << bits) - 1
    raw = b"".join((v & mask).to_bytes(8 * L, "little") for v in vals)
    return np.frombuffer(raw, dtype=np.uint64).reshape(len(vals), L).copy()


def digits32(vals: list[int], ndig: int) -> np.ndarray:
    """(n, ndig) uint64 array of the 32-bit digits of nonnegative ints."""
    raw = b"".join(v.to_bytes(4 * ndig, "little") for v in vals)
    return np.frombuffer(raw, dtype=np.uint32).reshape(len(vals), ndig).astype(np.uint64)


def residues(vals: list[int], primes) -> np.ndarray:
    """(np, n) v_i mod p_j for nonnegative ints v_i (crt_forward, rns.cpp:43-106)."""
    top = max((v.bit_length() for v in vals), default=1)
    nd = max(1, (top + 31) // 32)
    d = digits32(vals, nd)  # (n, nd)
    out = np.zeros((len(primes), len(vals)), np.uint64)
    for j, p in enumerate(int(x) for x in primes):
        acc = np.zeros(len(vals), np.uint64)
        w = 1
        pp = np.uint64(p)
        for m in range(nd):
            acc = (acc + (d[:, m] % pp) * np.uint64(w)) % pp
            w = (w << 32) % p
        out[j] = acc
    return out


def root_2n(p: int, n: int) -> int:
    """A primitive 2n-th root of unity mod p (p = 1 mod 2n)."""
    for c in range(2, 1 << 16):
        r = pow(c, (p - 1) // (2 * n), p)
        if pow(r, n, p) == p - 1:
            return r
    raise ValueError("no primitive 2n-th root")


def _powers(base: np.ndarray, P: np.ndarray, count: int) -> np.ndarray:
    """(rows, count) base^i mod P."""
    out = np.ones((len(base), count), np.uint64)
    if count > 1:
        out[:, 1] = base % P[:, 0]
    m = 2
    while m < count:
        step = np.array([pow(int(b), m, int(p)) for b, p in zip(base, P[:, 0])], np.uint64)
        k = min(m, count - m)
        out[:, m:m + k] = out[:, :k] * step[:, None] % P
        m *= 2
    return out


_REV: dict[int, np.ndarray] = {}


def _bit_reverse(n: int) -> np.ndarray:
    if n not in _REV:
        logn = n.bit_length() - 1
        rev = np.zeros(n, np.int64)
        for b in range(logn):
            rev |= ((np.arange(n) >> b) & 1) << (logn - 1 - b)
        _REV[n] = rev
    return _REV[n]


def _cyclic_ntt(x: np.ndarray, omega: np.ndarray, P: np.ndarray) -> np.ndarray:
    """Cyclic NTT of size n over rows (natural in, natural out)."""
    rows, n = x.shape
    x = x[:, _bit_reverse(n)].copy()
    h = 1
    while h < n:
        # twiddles omega^(n / (2h) * k), k < h
        wstep = np.array([pow(int(o), n // (2 * h), int(p)) for o, p in zip(omega, P[:, 0])],
                         np.uint64)
        tw = _powers(wstep, P, h)  # (rows, h)
        x = x.reshape(rows, n // (2 * h), 2, h)
        u = x[:, :, 0, :]
        v = x[:, :, 1, :] * tw[:, None, :] % P[:, :, None]
        x = np.stack([(u + v) % P[:, :, None], (u + P[:, :, None] - v) % P[:, :, None]], axis=2)
        x = x.reshape(rows, n)
        h *= 2
    return x


class NttPlan:
    """Negacyclic transforms mod one prime per row (psi = root_2n of the row's
    prime): fwd(a) = cyclic NTT of a psi^i, inv undoes it (natural order
    both ways; only the composition inv(fwd(a) fwd(b)) matters)."""

    def __init__(self, primes, n: int):
        self.P = np.asarray([int(p) for p in primes], np.uint64)[:, None]
        P = self.P
        self.n = n
        psi = np.array([root_2n(int(p), n) for p in P[:, 0]], np.uint64)
        self.tw = _powers(psi, P, n)
        self.omega = psi * psi % P[:, 0]
        self.oinv = np.array([pow(int(o), -1, int(p)) for o, p in zip(self.omega, P[:, 0])],
                             np.uint64)
        ninv = np.array([pow(n, -1, int(p)) for p in P[:, 0]], np.uint64)[:, None]
        psinv = np.array([pow(int(s), -1, int(p)) for s, p in zip(psi, P[:, 0])], np.uint64)
        self.itw = _powers(psinv, P, n) * ninv % P

    def fwd(self, a: np.ndarray) -> np.ndarray:
        a = np.asarray(a, np.uint64) % self.P
        return _cyclic_ntt(a * self.tw % self.P, self.omega, self.P)

    def inv(self, A: np.ndarray) -> np.ndarray:
        return _cyclic_ntt(np.asarray(A, np.uint64) % self.P, self.oinv, self.P) * self.itw % self.P


def negacyclic(a: np.ndarray, b: np.ndarray, primes) -> np.ndarray:
    """(rows, n) a * b mod (X^n + 1, p_r), rows of a / b reduced mod the row's
    prime (primes has one entry per row)."""
    plan = NttPlan(primes, np.asarray(a).shape[1])
    return plan.inv(plan.fwd(a) * plan.fwd(b) % plan.P)


def crt_hat_inverse(primes) -> np.ndarray:
    """((P / p_j) mod p_j)^-1 mod p_j: the t_j = x_j (P/p_j)^-1 factor the
    tensor-core iCRT / finisher operands carry (bigint_tc.cu)."""
    ps = [int(p) for p in primes]
    P = 1
    for p in ps:
        P *= p
    return np.array([pow((P // p) % p, -1, p) for p in ps], np.uint64)


def centred_lift(res: np.ndarray, primes) -> list[int]:
    """(np, n) residues -> the integers in (-P/2, P/2] (icrt, rns.cpp:132-190)."""
    ps = [int(p) for p in primes]
    P = 1
    for p in ps:
        P *= p
    coef = [(P // p) * pow((P // p) % p, -1, p) for p in ps]
    out = []
    cols = res.T.tolist()
    for col in cols:
        v = sum(int(r) * c for r, c in zip(col, coef)) % P
        out.append(v - P if v > P // 2 else v)
    return out
