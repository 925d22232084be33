/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference HE Mul path.
 * See hemul_oracle.h for the contract. This file is never linked into the
 * product (paper_2003_04510_b200/); the product fails loudly without its CUDA
 * library instead of falling back here.
 *
 * The restatement is deliberately simple: every modular product is a
 * 128-bit '%' (no Shoup tables), big integers are plain limb arrays, and the
 * iCRT folds below P by repeated subtraction. The residues and polynomials it
 * produces are canonical, hence identical to the reference's whatever
 * reduction tricks either side uses.
 */
#include "hemul_oracle.h"

#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)((u128)a * b % m);
}

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}

/* params.cpp:22-47: trial division by the first twelve primes, then
 * Miller-Rabin with those same twelve bases (deterministic below 2^64). */
static int is_prime(uint64_t n) {
  static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return 0;
  for (int i = 0; i < 12; ++i)
    if (n % bases[i] == 0) return n == bases[i];
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (int i = 0; i < 12; ++i) {
    uint64_t x = powmod(bases[i], d, n);
    if (x == 1 || x == n - 1) continue;
    int witness = 1;
    for (int r = 1; r < s && witness; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) witness = 0;
    }
    if (witness) return 0;
  }
  return 1;
}

/* params.cpp:49-54: psi = c^((p-1)/2n) for the smallest c >= 2 whose power
 * has psi^n == -1. */
static uint64_t root_2n(uint64_t p, uint64_t two_n) {
  for (uint64_t c = 2;; ++c) {
    const uint64_t psi = powmod(c, (p - 1) / two_n, p);
    if (powmod(psi, two_n / 2, p) == p - 1) return psi;
  }
}

int orc_prime_count(int bound_bits, int log_n) {
  /* params.cpp:76-79 with w64: 58 = guaranteed bits of each prime */
  return (bound_bits + log_n + 57) / 58;
}

int orc_generate_primes(int count, int log_n, uint64_t *primes,
                        uint64_t *roots) {
  const uint64_t two_n = (uint64_t)1 << (log_n + 1);
  const uint64_t hi = (uint64_t)1 << 60, lo = (uint64_t)1 << 57;
  int got = 0;
  /* params.cpp:99: largest c = 1 mod 2n at or below 2^60, then step -2n */
  for (uint64_t c = hi - (hi - 1) % two_n; got < count; c -= two_n) {
    if (c <= lo) return -1;
    if (!is_prime(c)) continue;
    primes[got] = c;
    if (roots) roots[got] = root_2n(c, two_n);
    ++got;
  }
  return got;
}

/* bit length of prod(primes[0..np)) */
static int product_bits(const uint64_t *primes, int np) {
  uint64_t *acc = calloc((size_t)np + 1, sizeof(uint64_t));
  int len = 1;
  acc[0] = 1;
  for (int j = 0; j < np; ++j) {
    uint64_t carry = 0;
    for (int k = 0; k < len; ++k) {
      const u128 t = (u128)acc[k] * primes[j] + carry;
      acc[k] = (uint64_t)t;
      carry = (uint64_t)(t >> 64);
    }
    if (carry) acc[len++] = carry;
  }
  int bits = (len - 1) * 64;
  uint64_t top = acc[len - 1];
  while (top) ++bits, top >>= 1;
  free(acc);
  return bits;
}

int orc_region_primes(int region, int log_q, int log_q_max, int log_n,
                      uint64_t *primes, uint64_t *roots, int cap) {
  /* heaan.cpp:132-135 (region 1: P1 >= 2^(2 log_q + log_n + 1)) and
   * heaan.cpp:139-143 (region 2: P2 >= 2^(log_q + 2 log_Q + log_n + 1)) */
  const int bound = region == 1 ? 2 * log_q + log_n + 1
                                : log_q + 2 * log_q_max + log_n + 1;
  int c = region == 1 ? orc_prime_count(2 * log_q, log_n)
                      : orc_prime_count(log_q + 2 * log_q_max, log_n);
  for (;; ++c) {
    uint64_t *ps = malloc(sizeof(uint64_t) * (size_t)c);
    uint64_t *rs = malloc(sizeof(uint64_t) * (size_t)c);
    if (orc_generate_primes(c, log_n, ps, roots ? rs : NULL) < 0) {
      free(ps), free(rs);
      return -1;
    }
    /* product >= 2^bound  <=>  bit length > bound */
    if (product_bits(ps, c) > bound) {
      for (int j = 0; j < c && j < cap; ++j) {
        primes[j] = ps[j];
        if (roots) roots[j] = rs[j];
      }
      free(ps), free(rs);
      return c;
    }
    free(ps), free(rs);
  }
}

static uint32_t bitrev(uint32_t i, int bits) {
  uint32_t r = 0;
  for (int b = 0; b < bits; ++b, i >>= 1) r = (r << 1) | (i & 1);
  return r;
}

void orc_ntt_tables(uint64_t p, uint64_t psi, int log_n, uint64_t *tw,
                    uint64_t *itw, uint64_t *n_inv) {
  /* params.cpp:160-178: tw[i] = psi^rev(i), itw[i] = psi^-rev(i) */
  const uint32_t n = 1u << log_n;
  const uint64_t psi_inv = powmod(psi, p - 2, p);
  uint64_t pw = 1, ipw = 1;
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t r = bitrev(i, log_n);
    tw[r] = pw;
    itw[r] = ipw;
    pw = mulmod(pw, psi, p);
    ipw = mulmod(ipw, psi_inv, p);
  }
  *n_inv = powmod(n % p, p - 2, p);
}

void orc_ntt_forward(uint64_t *x, int log_n, uint64_t p, const uint64_t *tw) {
  /* ntt.cpp:59-93 at radix 2: stage with m groups uses tw[m + g] on pairs
   * (j, j + t), t = n / 2m, Cooley-Tukey (ntt.cpp:11-33, exact branch) */
  const int n = 1 << log_n;
  int t = n;
  for (int m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (int g = 0; g < m; ++g) {
      const uint64_t w = tw[m + g];
      uint64_t *a = x + (size_t)2 * g * t;
      for (int j = 0; j < t; ++j) {
        const uint64_t u = a[j], v = mulmod(a[j + t], w, p);
        a[j] = u + v >= p ? u + v - p : u + v;
        a[j + t] = u >= v ? u - v : u + p - v;
      }
    }
  }
}

void orc_ntt_inverse(uint64_t *x, int log_n, uint64_t p, const uint64_t *itw,
                     uint64_t n_inv) {
  /* ntt.cpp:95-137 at radix 2: Gentleman-Sande from the widest groups down,
   * itw[m + g] on (u + v, (u - v) w) (ntt.cpp:36-57), then x n^-1 */
  const int n = 1 << log_n;
  for (int m = n >> 1, t = 1; m >= 1; m >>= 1, t <<= 1) {
    for (int g = 0; g < m; ++g) {
      const uint64_t w = itw[m + g];
      uint64_t *a = x + (size_t)2 * g * t;
      for (int j = 0; j < t; ++j) {
        const uint64_t u = a[j], v = a[j + t];
        a[j] = u + v >= p ? u + v - p : u + v;
        a[j + t] = mulmod(u >= v ? u - v : u + p - v, w, p);
      }
    }
  }
  for (int i = 0; i < n; ++i) x[i] = mulmod(x[i], n_inv, p);
}

void orc_crt(const uint64_t *poly, int n, int limbs, const uint64_t *primes,
             int np, uint64_t *out) {
  /* rns.cpp:43-106 (three_word_adc): sum_k a_{i,k} (2^64k mod p) in a
   * 192-bit accumulator, one reduction at the end. */
  uint64_t *pw = malloc(sizeof(uint64_t) * (size_t)limbs);
  for (int j = 0; j < np; ++j) {
    const uint64_t p = primes[j];
    const uint64_t beta = (uint64_t)(((u128)1 << 64) % p);
    const uint64_t beta2 = mulmod(beta, beta, p);
    pw[0] = 1 % p;
    for (int k = 1; k < limbs; ++k) pw[k] = mulmod(pw[k - 1], beta, p);
    for (int i = 0; i < n; ++i) {
      const uint64_t *c = poly + (size_t)i * limbs;
      u128 acc = 0;
      uint64_t top = 0;
      for (int k = 0; k < limbs; ++k) {
        const u128 m = (u128)c[k] * pw[k];
        acc += m;
        top += acc < m;
      }
      const uint64_t r = (uint64_t)((acc % p + (u128)mulmod(top % p, beta2, p)) % p);
      out[(size_t)j * n + i] = r;
    }
  }
  free(pw);
}

void orc_pointwise(const uint64_t *a, const uint64_t *b, int n,
                   const uint64_t *primes, int np, uint64_t *out) {
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < n; ++i) {
      const size_t ix = (size_t)j * n + i;
      out[ix] = mulmod(a[ix], b[ix], primes[j]);
    }
}

/* ---- small big-integer helpers on fixed-length limb arrays ---------------- */

static int big_cmp(const uint64_t *a, const uint64_t *b, int len) {
  for (int k = len - 1; k >= 0; --k)
    if (a[k] != b[k]) return a[k] < b[k] ? -1 : 1;
  return 0;
}

static void big_sub(uint64_t *a, const uint64_t *b, int len) { /* a -= b */
  uint64_t borrow = 0;
  for (int k = 0; k < len; ++k) {
    const uint64_t bk = b[k] + borrow;
    const uint64_t nb = (bk < borrow) || (a[k] < bk);
    a[k] -= bk;
    borrow = nb;
  }
}

/* q = a / d, returns remainder (len limbs) */
static uint64_t big_divw(uint64_t *q, const uint64_t *a, int len, uint64_t d) {
  u128 rem = 0;
  for (int k = len - 1; k >= 0; --k) {
    const u128 cur = (rem << 64) | a[k];
    q[k] = (uint64_t)(cur / d);
    rem = cur % d;
  }
  return (uint64_t)rem;
}

static uint64_t big_modw(const uint64_t *a, int len, uint64_t d) {
  u128 rem = 0;
  for (int k = len - 1; k >= 0; --k) rem = ((rem << 64) | a[k]) % d;
  return (uint64_t)rem;
}

void orc_icrt(const uint64_t *rns, int n, const uint64_t *primes, int np,
              int target_bits, uint64_t *out) {
  /* rns.cpp:132-190 + 235-290: t_j = x_j * (P/p_j)^-1 mod p_j;
   * acc = sum_j t_j * (P/p_j); fold below P (rns.cpp:148-158); residues above
   * floor(P/2) are the negative value acc - P (rns.cpp:159-167); reduce mod
   * 2^target_bits (rns.cpp:132-145). */
  const int pl = np + 1; /* P < 2^(60 np) fits np limbs; one guard */
  const int al = pl + 2;  /* the sum of np terms below np*P */
  const int tl = (target_bits + 63) / 64;
  uint64_t *P = calloc((size_t)al, 8), *hat = calloc((size_t)np * al, 8);
  uint64_t *halfP = calloc((size_t)al, 8), *acc = calloc((size_t)al, 8);
  uint64_t *inv = malloc(8 * (size_t)np);
  P[0] = 1;
  for (int j = 0; j < np; ++j) {
    uint64_t carry = 0;
    for (int k = 0; k < al; ++k) {
      const u128 t = (u128)P[k] * primes[j] + carry;
      P[k] = (uint64_t)t;
      carry = (uint64_t)(t >> 64);
    }
  }
  for (int j = 0; j < np; ++j) {
    uint64_t *h = hat + (size_t)j * al;
    big_divw(h, P, al, primes[j]);
    inv[j] = powmod(big_modw(h, al, primes[j]), primes[j] - 2, primes[j]);
  }
  for (int k = 0; k < al; ++k)
    halfP[k] = (P[k] >> 1) | (k + 1 < al ? P[k + 1] << 63 : 0);
  const uint64_t top_mask =
      target_bits % 64 ? ((uint64_t)1 << (target_bits % 64)) - 1 : ~(uint64_t)0;
  for (int i = 0; i < n; ++i) {
    memset(acc, 0, 8 * (size_t)al);
    for (int j = 0; j < np; ++j) {
      const uint64_t t = mulmod(rns[(size_t)j * n + i], inv[j], primes[j]);
      const uint64_t *h = hat + (size_t)j * al;
      uint64_t carry = 0;
      for (int k = 0; k < al; ++k) {
        const u128 s = (u128)t * h[k] + acc[k] + carry;
        acc[k] = (uint64_t)s;
        carry = (uint64_t)(s >> 64);
      }
    }
    while (big_cmp(acc, P, al) >= 0) big_sub(acc, P, al);
    uint64_t *o = out + (size_t)i * tl;
    if (big_cmp(acc, halfP, al) > 0) {
      /* negative: (acc - P) mod 2^T as a two's-complement wrap */
      uint64_t borrow = 0;
      for (int k = 0; k < tl; ++k) {
        const uint64_t a = k < al ? acc[k] : 0, b = k < al ? P[k] : 0;
        const uint64_t bk = b + borrow;
        const uint64_t nb = (bk < borrow) || (a < bk);
        o[k] = a - bk;
        borrow = nb;
      }
    } else {
      for (int k = 0; k < tl; ++k) o[k] = k < al ? acc[k] : 0;
    }
    o[tl - 1] &= top_mask;
  }
  free(P), free(hat), free(halfP), free(acc), free(inv);
}

static uint64_t mask_top(int log_q) {
  return log_q % 64 ? ((uint64_t)1 << (log_q % 64)) - 1 : ~(uint64_t)0;
}

void orc_poly_add(const uint64_t *a, const uint64_t *b, int n, int log_q,
                  uint64_t *out) {
  /* poly.cpp:46-70 */
  const int L = (log_q + 63) / 64;
  for (int i = 0; i < n; ++i) {
    uint64_t carry = 0;
    for (int k = 0; k < L; ++k) {
      const size_t ix = (size_t)i * L + k;
      const u128 s = (u128)a[ix] + b[ix] + carry;
      out[ix] = (uint64_t)s;
      carry = (uint64_t)(s >> 64);
    }
    out[(size_t)i * L + L - 1] &= mask_top(log_q);
  }
}

void orc_poly_sub(const uint64_t *a, const uint64_t *b, int n, int log_q,
                  uint64_t *out) {
  /* poly.cpp:73-91 */
  const int L = (log_q + 63) / 64;
  for (int i = 0; i < n; ++i) {
    uint64_t borrow = 0;
    for (int k = 0; k < L; ++k) {
      const size_t ix = (size_t)i * L + k;
      const uint64_t bk = b[ix] + borrow;
      const uint64_t nb = (bk < borrow) || (a[ix] < bk);
      out[ix] = a[ix] - bk;
      borrow = nb;
    }
    out[(size_t)i * L + L - 1] &= mask_top(log_q);
  }
}

void orc_shift_right(const uint64_t *a, int n, int log_q, int bits,
                     uint64_t *out) {
  /* poly.cpp:98-115: s = v + 2^(bits-1); if s >= 2^log_q then s -= 2^log_q;
   * out = s >> bits, a residue mod 2^(log_q - bits). */
  const int L = (log_q + 63) / 64, Lo = (log_q - bits + 63) / 64;
  uint64_t *s = malloc(8 * ((size_t)L + 1));
  for (int i = 0; i < n; ++i) {
    const uint64_t *v = a + (size_t)i * L;
    uint64_t carry = 0;
    for (int k = 0; k <= L; ++k) {
      const uint64_t add = (k == (bits - 1) / 64) ? (uint64_t)1 << ((bits - 1) % 64) : 0;
      const u128 t = (u128)(k < L ? v[k] : 0) + add + carry;
      s[k] = (uint64_t)t;
      carry = (uint64_t)(t >> 64);
    }
    /* wrap mod 2^log_q: clear every bit at or above log_q */
    for (int k = log_q / 64; k <= L; ++k) {
      if (k == log_q / 64)
        s[k] &= mask_top(log_q) == ~(uint64_t)0 ? 0 : mask_top(log_q);
      else
        s[k] = 0;
    }
    uint64_t *o = out + (size_t)i * Lo;
    const int wq = bits / 64, bq = bits % 64;
    for (int k = 0; k < Lo; ++k) {
      const uint64_t lo = wq + k <= L ? s[wq + k] : 0;
      const uint64_t hi = wq + k + 1 <= L ? s[wq + k + 1] : 0;
      o[k] = bq ? (lo >> bq) | (hi << (64 - bq)) : lo;
    }
    o[Lo - 1] &= mask_top(log_q - bits);
  }
  free(s);
}

/* pm_prepare (polymul.cpp:7-20): CRT + forward NTT per prime row */
static void prepare(const uint64_t *poly, int n, int log_n, int limbs,
                    const uint64_t *primes, const uint64_t *tw, int np,
                    uint64_t *out) {
  orc_crt(poly, n, limbs, primes, np, out);
  for (int j = 0; j < np; ++j)
    orc_ntt_forward(out + (size_t)j * n, log_n, primes[j], tw + (size_t)j * n);
}

/* pm_finish (polymul.cpp:29-37): inverse NTT per row + iCRT */
static void finish(uint64_t *rns, int n, int log_n, const uint64_t *primes,
                   const uint64_t *itw, const uint64_t *ninv, int np,
                   int target_bits, uint64_t *out) {
  for (int j = 0; j < np; ++j)
    orc_ntt_inverse(rns + (size_t)j * n, log_n, primes[j], itw + (size_t)j * n,
                    ninv[j]);
  orc_icrt(rns, n, primes, np, target_bits, out);
}

int orc_he_mul(int log_n, int log_p, int log_q_max, int log_q, int c2_log_q,
               const uint64_t *c1ax, const uint64_t *c1bx,
               const uint64_t *c2ax, const uint64_t *c2bx,
               const uint64_t *evk_ax, const uint64_t *evk_bx,
               uint64_t *out_ax, uint64_t *out_bx) {
  /* heaan.cpp:341-345: validation order and error kinds */
  if (log_q != c2_log_q) return 2;
  if (log_q - log_p < log_p) return 3;
  const int n = 1 << log_n, L = (log_q + 63) / 64;
  const int log_Q = log_q_max, L2 = (log_q + log_Q + 63) / 64;
  const int Le = (2 * log_Q + 63) / 64;
  const int np1 = orc_region_primes(1, log_q, log_Q, log_n, NULL, NULL, 0);
  const int np2 = orc_region_primes(2, log_q, log_Q, log_n, NULL, NULL, 0);
  if (np1 < 0 || np2 < 0) return 1;
  const int npm = np1 > np2 ? np1 : np2;
  uint64_t *pr = malloc(8 * (size_t)npm), *rt = malloc(8 * (size_t)npm);
  uint64_t *tw1 = malloc(8 * (size_t)np1 * n), *itw1 = malloc(8 * (size_t)np1 * n);
  uint64_t *tw2 = malloc(8 * (size_t)np2 * n), *itw2 = malloc(8 * (size_t)np2 * n);
  uint64_t *p1 = malloc(8 * (size_t)np1), *p2 = malloc(8 * (size_t)np2);
  uint64_t *ni1 = malloc(8 * (size_t)np1), *ni2 = malloc(8 * (size_t)np2);
  orc_region_primes(1, log_q, log_Q, log_n, pr, rt, npm);
  for (int j = 0; j < np1; ++j) {
    p1[j] = pr[j];
    orc_ntt_tables(pr[j], rt[j], log_n, tw1 + (size_t)j * n, itw1 + (size_t)j * n, &ni1[j]);
  }
  orc_region_primes(2, log_q, log_Q, log_n, pr, rt, npm);
  for (int j = 0; j < np2; ++j) {
    p2[j] = pr[j];
    orc_ntt_tables(pr[j], rt[j], log_n, tw2 + (size_t)j * n, itw2 + (size_t)j * n, &ni2[j]);
  }
  const size_t r1 = (size_t)np1 * n, r2 = (size_t)np2 * n, pq = (size_t)n * L;
  uint64_t *fa = malloc(8 * r1), *fb = malloc(8 * r1);
  uint64_t *d0 = malloc(8 * pq), *d1 = malloc(8 * pq), *d2 = malloc(8 * pq);
  uint64_t *s1 = malloc(8 * pq), *s2 = malloc(8 * pq);
  /* region 1 (heaan.cpp:372-394): d0 = bx1 bx2, d2 = ax1 ax2,
   * d1 = (ax1 + bx1)(ax2 + bx2) - d0 - d2, all mod 2^log_q */
  prepare(c1bx, n, log_n, L, p1, tw1, np1, fa);
  prepare(c2bx, n, log_n, L, p1, tw1, np1, fb);
  orc_pointwise(fa, fb, n, p1, np1, fa);
  finish(fa, n, log_n, p1, itw1, ni1, np1, log_q, d0);
  prepare(c1ax, n, log_n, L, p1, tw1, np1, fa);
  prepare(c2ax, n, log_n, L, p1, tw1, np1, fb);
  orc_pointwise(fa, fb, n, p1, np1, fa);
  finish(fa, n, log_n, p1, itw1, ni1, np1, log_q, d2);
  orc_poly_add(c1ax, c1bx, n, log_q, s1);
  orc_poly_add(c2ax, c2bx, n, log_q, s2);
  prepare(s1, n, log_n, L, p1, tw1, np1, fa);
  prepare(s2, n, log_n, L, p1, tw1, np1, fb);
  orc_pointwise(fa, fb, n, p1, np1, fa);
  finish(fa, n, log_n, p1, itw1, ni1, np1, log_q, d1);
  orc_poly_sub(d1, d0, n, log_q, d1);
  orc_poly_sub(d1, d2, n, log_q, d1);
  free(fa), free(fb), free(s1), free(s2);
  /* region 2 (heaan.cpp:396-402): key switching of d2 against the evk forms
   * (heaan.cpp:152-167, CRT over 2 log_Q-bit inputs), ModDown by R_logQ */
  uint64_t *fd = malloc(8 * r2), *fe = malloc(8 * r2), *pr2 = malloc(8 * r2);
  uint64_t *ks = malloc(8 * (size_t)n * L2), *ksq = malloc(8 * pq);
  uint64_t *c3 = malloc(8 * pq);
  prepare(d2, n, log_n, L, p2, tw2, np2, fd);
  const uint64_t *evk[2] = {evk_ax, evk_bx};
  const uint64_t *dd[2] = {d1, d0};
  uint64_t *outs[2] = {out_ax, out_bx};
  for (int c = 0; c < 2; ++c) {
    prepare(evk[c], n, log_n, Le, p2, tw2, np2, fe);
    orc_pointwise(fd, fe, n, p2, np2, pr2);
    finish(pr2, n, log_n, p2, itw2, ni2, np2, log_q + log_Q, ks);
    orc_shift_right(ks, n, log_q + log_Q, log_Q, ksq);
    /* heaan.cpp:404-409: c3 = d + ks_q, then rescale by log_p
     * (heaan.cpp:328-337) */
    orc_poly_add(dd[c], ksq, n, log_q, c3);
    orc_shift_right(c3, n, log_q, log_p, outs[c]);
  }
  free(fd), free(fe), free(pr2), free(ks), free(ksq), free(c3);
  free(d0), free(d1), free(d2);
  free(pr), free(rt), free(tw1), free(itw1), free(tw2), free(itw2);
  free(p1), free(p2), free(ni1), free(ni2);
  return 0;
}

uint64_t orc_digest(int log_q, int n, const uint64_t *ax, const uint64_t *bx) {
  /* bench.cpp:35-47: FNV-1a 64 over log_q, then ax words, then bx words,
   * each word's bytes little-endian */
  const size_t words = (size_t)n * ((log_q + 63) / 64);
  uint64_t h = 1469598103934665603ull;
  uint64_t v = (uint64_t)log_q;
  for (int k = 0; k < 8; ++k) h = (h ^ ((v >> (8 * k)) & 0xff)) * 1099511628211ull;
  for (size_t i = 0; i < 2 * words; ++i) {
    v = i < words ? ax[i] : bx[i - words];
    for (int k = 0; k < 8; ++k) h = (h ^ ((v >> (8 * k)) & 0xff)) * 1099511628211ull;
  }
  return h;
}
