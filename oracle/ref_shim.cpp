// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the reference library compiled from the
// read-only sources under /root/reference/proj/core (see oracle/Makefile; the
// namespace is renamed hemul -> hemul_ref on the command line). tests/ and
// bench.py (cpu_baseline / --impl reference) load oracle/_ref/libhemul_ref.so
// through ctypes to
//   * regenerate the seed-7 bench-protocol inputs and digests
//     (proj/core/src/bench.cpp:49-124),
//   * run Scheme::he_mul on arbitrary inputs (proj/core/src/heaan.cpp:339-410),
//   * expose the per-stage kernels (CRT / NTT / pointwise / iCRT) on the same
//     level tables Scheme::level builds (proj/core/src/heaan.cpp:119-169),
// so every GPU stage can be compared residue for residue.
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "hemul/bench.hpp"
#include "hemul/heaan.hpp"
#include "hemul/io.hpp"
#include "hemul/ntt.hpp"
#include "hemul/params.hpp"
#include "hemul/poly.hpp"
#include "hemul/polymul.hpp"
#include "hemul/rns.hpp"
#include "hemul/rng.hpp"
#include "hemul/thread_pool.hpp"

using namespace hemul;  // renamed to hemul_ref by -Dhemul=hemul_ref

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

BigPoly poly_from(const uint64_t* src, int n, int log_q) {
  BigPoly p = make_poly(n, log_q, WordSize::w64);
  std::memcpy(p.data.data(), src, sizeof(uint64_t) * p.data.size());
  return p;
}

void poly_to(const BigPoly& p, uint64_t* dst) {
  std::memcpy(dst, p.data.data(), sizeof(uint64_t) * p.data.size());
}

// Mirrors the prime-set construction of Scheme::level (heaan.cpp:132-147).
struct RegionTables {
  PrimeSet ps;
  CrtTables crt;
  NttTables ntt;
  IcrtTables icrt;
};

std::unique_ptr<RegionTables> build_region(int region, int log_q, int log_q_max,
                                           int log_n, int crt_bits) {
  auto t = std::make_unique<RegionTables>();
  const WordSize w = WordSize::w64;
  int c = 0;
  int bound = 0, target_bits = 0;
  if (region == 1) {
    c = region1_prime_count(log_q, log_n, w);
    bound = 2 * log_q + log_n + 1;
    target_bits = log_q;
  } else {
    c = region2_prime_count(log_q, log_q_max, log_n, w);
    bound = log_q + 2 * log_q_max + log_n + 1;
    target_bits = log_q + log_q_max;
  }
  t->ps = generate_primes(c, log_n, w);
  while (bigint_cmp(t->ps.product, bigint_pow2(bound, w)) < 0)
    t->ps = generate_primes(++c, log_n, w);
  t->crt = make_crt_tables(t->ps, crt_bits > 0 ? crt_bits : log_q);
  t->ntt = make_ntt_tables(t->ps, log_n);
  t->icrt = make_icrt_tables(t->ps, bigint_pow2(target_bits, w), w);
  return t;
}

PmContext ctx_of(const RegionTables& t) {
  PmContext c;
  c.ps = &t.ps;
  c.crt = &t.crt;
  c.ntt = &t.ntt;
  c.icrt = &t.icrt;
  return c;
}

}  // namespace

namespace {

// FNV-1a over every field of the lower-level tables of one prime set
// (params.hpp: PrimeSet, CrtTables, NttTables, IcrtTables); the same routine
// is in tests/cpp/dropin_check.cpp and oracle/ref_shim.cpp.
struct TableHash {
  uint64_t h = 1469598103934665603ull;
  void word(uint64_t v) {
    for (int k = 0; k < 8; ++k) h = (h ^ ((v >> (8 * k)) & 0xff)) * 1099511628211ull;
  }
  void words(const std::vector<uint64_t>& v) {
    word(v.size());
    for (uint64_t x : v) word(x);
  }
  void pairs(const std::vector<ShoupPair>& v) {
    word(v.size());
    for (const ShoupPair& s : v) {
      word(s.value);
      word(s.quotient);
    }
  }
};

uint64_t table_digest(int np, int log_n, int log_q, bool w32) {
  const WordSize w = w32 ? WordSize::w32 : WordSize::w64;
  const PrimeSet ps = generate_primes(np, log_n, w);
  const CrtTables ct = make_crt_tables(ps, log_q);
  const NttTables nt = make_ntt_tables(ps, log_n);
  const IcrtTables it = make_icrt_tables(ps, bigint_pow2(log_q, w), w);
  TableHash t;
  t.word(ps.two_n);
  t.words(ps.primes);
  t.words(ps.roots);
  t.pairs(ps.pair_one);
  t.pairs(ps.pair_beta);
  t.pairs(ps.pair_beta2);
  t.words(ps.product);
  t.word(ct.np);
  t.word(ct.q_limbs);
  t.pairs(ct.pow_beta);
  t.word(nt.log_n);
  t.word(nt.n);
  t.pairs(nt.tw);
  t.pairs(nt.itw);
  t.pairs(nt.n_inv);
  t.word(it.np);
  t.word(it.p_limbs);
  t.pairs(it.inv_p);
  t.words(it.p_div_p);
  t.words(it.p_div_p_t);
  t.words(it.big_p);
  t.words(it.half_p);
  t.words(it.neg_p_mod);
  for (const auto& m : it.p_multiples) t.words(m);
  t.words(it.target);
  t.word(it.target_pow2);
  t.word(it.target_log2);
  t.word(it.accum_words);
  return t.h;
}

}  // namespace

extern "C" {

// save_params (io.cpp:54-70) of make_params(log_p, depth, w64, log_n_override)
int ref_save_params(const char* path, int log_p, int depth, int log_n_override) {
  try {
    save_params(path, make_params(log_p, depth, WordSize::w64, log_n_override));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

uint64_t ref_table_digest(int np, int log_n, int log_q, int w32) {
  try {
    return table_digest(np, log_n, log_q, w32 != 0);
  } catch (const std::exception& e) {
    return (void)fail(e, 1), 0;
  }
}

const char* ref_last_error() { return g_err.c_str(); }

// make_params (params.cpp:64-74): out = {log_n, n, log_q_max}
int ref_make_params(int log_p, int depth, int log_n_override, int* out) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    out[0] = p.log_n;
    out[1] = p.n;
    out[2] = p.log_q_max;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Prime set of one region at one level (heaan.cpp:132-143); returns the count
// (or -1), writes up to cap primes and roots.
int ref_level_primes(int region, int log_q, int log_q_max, int log_n,
                     uint64_t* primes, uint64_t* roots, int cap) {
  try {
    auto t = build_region(region, log_q, log_q_max, log_n, 0);
    const int np = static_cast<int>(t->ps.primes.size());
    for (int j = 0; j < np && j < cap; ++j) {
      primes[j] = t->ps.primes[j];
      if (roots) roots[j] = t->ps.roots[j];
    }
    return np;
  } catch (const std::exception& e) {
    return (void)fail(e, 1), -1;
  }
}

// Bench-protocol inputs (bench.cpp:60-67): seed -> keygen, two random
// messages, encode, encrypt. Buffers: ct polys n*ceil(log_q_max/64), evk polys
// n*ceil(2 log_q_max/64).
int ref_bench_inputs(int log_p, int depth, int log_n_override, uint64_t seed,
                     uint64_t* c1ax, uint64_t* c1bx, uint64_t* c2ax,
                     uint64_t* c2bx, uint64_t* evk_ax, uint64_t* evk_bx,
                     int* sk_out) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    Scheme scheme(p);
    Rng rng(seed);
    const int ns = std::min(64, p.n / 2);
    auto msg = [&](Rng& r) {
      Message m;
      m.slots.resize(ns);
      for (auto& s : m.slots) {
        const double re = static_cast<double>(r.next() >> 11) * 0x1p-53 * 2 - 1;
        const double im = static_cast<double>(r.next() >> 11) * 0x1p-53 * 2 - 1;
        s = {re, im};
      }
      return m;
    };
    const KeySet keys = scheme.keygen(rng);
    const Plaintext t1 = scheme.encode(msg(rng));
    const Plaintext t2 = scheme.encode(msg(rng));
    const Ciphertext c1 = scheme.encrypt(t1, keys.pk, rng);
    const Ciphertext c2 = scheme.encrypt(t2, keys.pk, rng);
    poly_to(c1.ax, c1ax);
    poly_to(c1.bx, c1bx);
    poly_to(c2.ax, c2ax);
    poly_to(c2.bx, c2bx);
    poly_to(keys.evk.ax, evk_ax);
    poly_to(keys.evk.bx, evk_bx);
    if (sk_out)
      for (int i = 0; i < p.n; ++i) sk_out[i] = keys.sk.s[i];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Scheme::he_mul on caller inputs at modulus log_q (heaan.cpp:339-410).
// Returns 0, 2 (invalid_argument), 3 (runtime_error).
int ref_he_mul(int log_p, int depth, int log_n_override, int log_q,
               const uint64_t* c1ax, const uint64_t* c1bx, const uint64_t* c2ax,
               const uint64_t* c2bx, int c2_log_q, const uint64_t* evk_ax,
               const uint64_t* evk_bx, uint64_t* out_ax, uint64_t* out_bx,
               int threads, int radix_log) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    std::unique_ptr<ThreadPool> pool;
    if (threads > 1) pool = std::make_unique<ThreadPool>(threads);
    Scheme scheme(p, pool.get());
    scheme.options().ntt.radix_log = radix_log > 0 ? radix_log : 1;
    Ciphertext c1, c2;
    c1.ax = poly_from(c1ax, p.n, log_q);
    c1.bx = poly_from(c1bx, p.n, log_q);
    c1.log_q = log_q;
    c2.ax = poly_from(c2ax, p.n, c2_log_q);
    c2.bx = poly_from(c2bx, p.n, c2_log_q);
    c2.log_q = c2_log_q;
    EvalKey evk;
    evk.ax = poly_from(evk_ax, p.n, 2 * p.log_q_max);
    evk.bx = poly_from(evk_bx, p.n, 2 * p.log_q_max);
    const Ciphertext out = scheme.he_mul(c1, c2, evk);
    poly_to(out.ax, out_ax);
    poly_to(out.bx, out_bx);
    return 0;
  } catch (const std::invalid_argument& e) {
    return fail(e, 2);
  } catch (const std::runtime_error& e) {
    return fail(e, 3);
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// run_he_mul_bench (bench.cpp:49-124). ms_out = {crt, ntt, intt, icrt, extra,
// total_mean, total_median}.
int ref_run_bench(int log_p, int depth, int log_n_override, uint64_t seed,
                  int reps, int threads, int radix_log, double* ms_out,
                  uint64_t* digest) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    BenchConfig cfg;
    cfg.seed = seed;
    cfg.reps = reps;
    cfg.threads = threads;
    cfg.radix_log = radix_log > 0 ? radix_log : 1;
    std::unique_ptr<ThreadPool> pool;
    if (threads > 1) pool = std::make_unique<ThreadPool>(threads);
    const BenchReport r = run_he_mul_bench(p, cfg, pool.get());
    if (ms_out) {
      ms_out[0] = r.crt_ms;
      ms_out[1] = r.ntt_ms;
      ms_out[2] = r.intt_ms;
      ms_out[3] = r.icrt_ms;
      ms_out[4] = r.extra_ms;
      ms_out[5] = r.total_ms;
      ms_out[6] = r.total_median_ms;
    }
    if (digest) *digest = r.result_digest;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// The CPU baseline: one Scheme, level + evk forms warmed outside the timing
// (bench.cpp:68-69), then `reps` timed he_mul calls on random ciphertexts and
// a random evk (uniform_bits, rng.hpp:30-41) at the fresh modulus.
// ms_out[r] = wall milliseconds of rep r. Returns the output digest.
int ref_time_he_mul(int log_p, int depth, int log_n_override, uint64_t seed, int reps,
                    int threads, int radix_log, double* ms_out, uint64_t* digest) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    std::unique_ptr<ThreadPool> pool;
    if (threads > 1) pool = std::make_unique<ThreadPool>(threads);
    Scheme scheme(p, pool.get());
    scheme.options().ntt.radix_log = radix_log > 0 ? radix_log : 1;
    Rng rng(seed);
    auto rnd = [&](int bits) {
      BigPoly a = make_poly(p.n, bits, WordSize::w64);
      for (int i = 0; i < p.n; ++i) poly_set(a, i, rng.uniform_bits(bits, WordSize::w64));
      return a;
    };
    Ciphertext c1, c2;
    c1.ax = rnd(p.log_q_max);
    c1.bx = rnd(p.log_q_max);
    c2.ax = rnd(p.log_q_max);
    c2.bx = rnd(p.log_q_max);
    c1.log_q = c2.log_q = p.log_q_max;
    EvalKey evk;
    evk.ax = rnd(2 * p.log_q_max);
    evk.bx = rnd(2 * p.log_q_max);
    scheme.warm_level(p.log_q_max, &evk);
    Ciphertext out;
    for (int r = 0; r < reps; ++r) {
      const auto t0 = std::chrono::steady_clock::now();
      out = scheme.he_mul(c1, c2, evk);
      const auto t1 = std::chrono::steady_clock::now();
      ms_out[r] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
    if (digest) *digest = ciphertext_digest(out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Scheme::counters after one he_mul on the bench-protocol inputs (seed):
// out[5 * 4] = {mul, adc, modmul, addsub} per stage (counters.hpp:13-31).
// four_products / periodic select SchemeOptions (periodic: period 4).
int ref_counters(int log_p, int depth, int log_n_override, uint64_t seed, int four_products,
                 int periodic, uint64_t* out) {
  try {
    const Params p = make_params(log_p, depth, WordSize::w64, log_n_override);
    Scheme scheme(p);
    scheme.options().four_products = four_products != 0;
    if (periodic) {
      scheme.options().strategy.kind = AccumKind::periodic_mod;
      scheme.options().strategy.period = 4;
    }
    Rng rng(seed);
    const KeySet keys = scheme.keygen(rng);
    Message m;
    m.slots.assign(std::min(8, p.n / 2), {0.5, -0.25});
    const Ciphertext c1 = scheme.encrypt(scheme.encode(m), keys.pk, rng);
    const Ciphertext c2 = scheme.encrypt(scheme.encode(m), keys.pk, rng);
    scheme.warm_level(p.log_q_max, &keys.evk);
    scheme.counters.reset();
    scheme.he_mul(c1, c2, keys.evk);
    for (int s = 0; s < 5; ++s) {
      const OpCounts& c = scheme.counters.stage[s];
      out[4 * s + 0] = c.mul;
      out[4 * s + 1] = c.adc;
      out[4 * s + 2] = c.modmul;
      out[4 * s + 3] = c.addsub;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// ciphertext_digest (bench.cpp:35-47) over caller buffers.
uint64_t ref_digest(int log_q, int n, const uint64_t* ax, const uint64_t* bx) {
  Ciphertext c;
  c.ax = poly_from(ax, n, log_q);
  c.bx = poly_from(bx, n, log_q);
  c.log_q = log_q;
  return ciphertext_digest(c);
}

// --- stage kernels on one region's level tables -----------------------------

// pm_prepare (polymul.cpp:7-20): CRT of an n x ceil(in_bits/64) BigPoly into
// the region's primes, then forward NTT. out: np x n prime-major.
// stop_after_crt=1 returns the CRT residues without the NTT.
int ref_prepare(int region, int log_q, int log_q_max, int log_n, int in_bits,
                const uint64_t* poly, uint64_t* out, int stop_after_crt) {
  try {
    auto t = build_region(region, log_q, log_q_max, log_n, in_bits);
    const BigPoly a = poly_from(poly, 1 << log_n, in_bits);
    RnsMatrix m = crt_forward(a, t->ps, t->crt, AccumStrategy{},
                              Layout::prime_major);
    if (!stop_after_crt) ntt_forward(m, t->ps, t->ntt);
    std::memcpy(out, m.data.data(), sizeof(uint64_t) * m.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// Forward (inverse=0) or inverse NTT in place over np x n prime-major rows.
// bench_ntt.cpp:10-27 protocol widened to the C2 sweep:
// generate_primes(np, log_n, w64), residues Rng(3).below(p_j), `reps` timed
// ntt_forward / ntt_inverse calls on a fresh copy each (copy untimed), on
// `threads` threads (ThreadPool) at NTT radix 2^radix_log.
int ref_time_ntt(int log_n, int np, int threads, int radix_log, int reps, int inverse,
                 double* ms_out) {
  try {
    const PrimeSet ps = generate_primes(np, log_n, WordSize::w64);
    const NttTables nt = make_ntt_tables(ps, log_n);
    const int n = 1 << log_n;
    Rng rng(3);
    RnsMatrix m = make_rns(np, n, Layout::prime_major);
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < n; ++i) m.at(j, i) = rng.below(ps.primes[j]);
    std::unique_ptr<ThreadPool> pool;
    if (threads > 1) pool = std::make_unique<ThreadPool>(threads);
    NttOptions opt;
    opt.radix_log = radix_log > 0 ? radix_log : 1;
    for (int r = 0; r < reps; ++r) {
      RnsMatrix copy = m;
      const auto t0 = std::chrono::steady_clock::now();
      if (inverse)
        ntt_inverse(copy, ps, nt, opt, pool.get());
      else
        ntt_forward(copy, ps, nt, opt, pool.get());
      const auto t1 = std::chrono::steady_clock::now();
      ms_out[r] = std::chrono::duration<double, std::milli>(t1 - t0).count();
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_ntt(int region, int log_q, int log_q_max, int log_n, uint64_t* data,
            int inverse) {
  try {
    auto t = build_region(region, log_q, log_q_max, log_n, 0);
    RnsMatrix m = make_rns(static_cast<int>(t->ps.primes.size()), 1 << log_n,
                           Layout::prime_major);
    std::memcpy(m.data.data(), data, sizeof(uint64_t) * m.data.size());
    if (inverse)
      ntt_inverse(m, t->ps, t->ntt);
    else
      ntt_forward(m, t->ps, t->ntt);
    std::memcpy(data, m.data.data(), sizeof(uint64_t) * m.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// pm_finish (polymul.cpp:29-37): iNTT + reordered iCRT of an np x n product to
// a BigPoly mod the region target (2^log_q or 2^(log_q+log_q_max)).
// skip_intt=1 runs only the iCRT.
int ref_finish(int region, int log_q, int log_q_max, int log_n,
               const uint64_t* rns, uint64_t* out, int skip_intt) {
  try {
    auto t = build_region(region, log_q, log_q_max, log_n, 0);
    RnsMatrix m = make_rns(static_cast<int>(t->ps.primes.size()), 1 << log_n,
                           Layout::prime_major);
    std::memcpy(m.data.data(), rns, sizeof(uint64_t) * m.data.size());
    BigPoly r;
    if (skip_intt)
      r = icrt_reordered(m, t->ps, t->icrt);
    else
      r = pm_finish(std::move(m), ctx_of(*t));
    poly_to(r, out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// rns_pointwise_mul (rns.cpp:360-371).
int ref_pointwise(int region, int log_q, int log_q_max, int log_n,
                  const uint64_t* a, const uint64_t* b, uint64_t* out) {
  try {
    auto t = build_region(region, log_q, log_q_max, log_n, 0);
    const int np = static_cast<int>(t->ps.primes.size());
    RnsMatrix ma = make_rns(np, 1 << log_n, Layout::prime_major), mb = ma, r;
    std::memcpy(ma.data.data(), a, sizeof(uint64_t) * ma.data.size());
    std::memcpy(mb.data.data(), b, sizeof(uint64_t) * mb.data.size());
    rns_pointwise_mul(r, ma, mb, t->ps);
    std::memcpy(out, r.data.data(), sizeof(uint64_t) * r.data.size());
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// poly_shift_right (poly.cpp:98-115).
int ref_shift_right(int n, int log_q, int bits, const uint64_t* a,
                    uint64_t* out) {
  try {
    const BigPoly r = poly_shift_right(poly_from(a, n, log_q), bits);
    poly_to(r, out);
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

}  // extern "C"
