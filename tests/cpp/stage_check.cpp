// Restated lower-level tests of the reference (proj/tests/test_ntt.cpp,
// test_rns.cpp, test_polymul.cpp, test_arith.cpp) compiled against the
// drop-in headers (include/hemul/{word,params,rns,ntt,polymul}.hpp) and run
// on the GPU through libhemul_gpu.so. doctest and GMP are not in this image:
// CHECK counts failures, and the GMP oracles are restated with the drop-in
// BigInt arithmetic (independent of the GPU kernels under test).
//
//   stage_check [--quick]     prints "failures <k>" and exits 1 on any failure
#include <cstdio>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "hemul/polymul.hpp"
#include "hemul/rng.hpp"

using namespace hemul;

namespace {

int g_failures = 0, g_checks = 0;
std::string g_case;

#define CHECK(cond)                                                                      \
  do {                                                                                   \
    ++g_checks;                                                                          \
    if (!(cond)) {                                                                       \
      if (++g_failures <= 20)                                                            \
        std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); \
    }                                                                                    \
  } while (0)

template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

void run_case(const char* name, const std::function<void()>& body) {
  g_case = name;
  const int before = g_failures;
  try {
    body();
  } catch (const std::exception& e) {
    ++g_failures;
    std::printf("FAIL [%s] exception: %s\n", name, e.what());
  }
  std::printf("%s %s\n", g_failures == before ? "ok  " : "FAIL", name);
}

// test_ntt.cpp:12-27
std::vector<uint64_t> negacyclic_mod_p(const std::vector<uint64_t>& a,
                                       const std::vector<uint64_t>& b, uint64_t p) {
  const int n = static_cast<int>(a.size());
  std::vector<uint64_t> r(n, 0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const uint64_t t = mulmod_u64(a[i], b[j], p);
      if (i + j < n)
        r[i + j] = add_mod(r[i + j], t, p);
      else
        r[i + j - n] = sub_mod(r[i + j - n], t, p);
    }
  return r;
}

RnsMatrix random_matrix(const PrimeSet& ps, int n, Rng& rng) {
  const int np = static_cast<int>(ps.primes.size());
  RnsMatrix m = make_rns(np, n, Layout::prime_major);
  for (int j = 0; j < np; ++j)
    for (int i = 0; i < n; ++i) m.at(j, i) = rng.below(ps.primes[j]);
  return m;
}

BigPoly random_poly(int n, int log_q, Rng& rng) {
  BigPoly a = make_poly(n, log_q, WordSize::w64);
  for (auto& x : a.data) x = rng.next();
  for (int i = 0; i < n; ++i) poly_set(a, i, poly_get(a, i));  // mask the top limb
  return a;
}

// signed negacyclic product mod 2^log_q (the GMP oracle of
// test_polymul.cpp:19-43, restated with BigInt)
BigPoly exact_negacyclic(const BigPoly& a, const BigPoly& b) {
  const WordSize w = WordSize::w64;
  const int n = a.n;
  const BigInt q = bigint_pow2(a.log_q, w);
  BigPoly r = make_poly(n, a.log_q, w);
  for (int k = 0; k < n; ++k) {
    BigInt plus = {}, minus = {};
    for (int i = 0; i < n; ++i) {
      const int j = k - i;
      const BigInt t = bigint_mul(poly_get(a, i), poly_get(b, (j + n) % n), w);
      BigInt& acc = j >= 0 ? plus : minus;
      BigInt s;
      const uint64_t c = bigint_add(s, acc, t, w);
      if (c) s.push_back(c);
      acc = std::move(s);
    }
    BigInt u = bigint_mod(plus, q, w), v = bigint_mod(minus, q, w), d;
    if (bigint_cmp(u, v) < 0) {
      BigInt s;
      bigint_add(s, u, q, w);
      u = std::move(s);
    }
    bigint_sub(d, u, v, w);
    poly_set(r, k, d);
  }
  return r;
}

PrimeSet p17_set() {  // test_ntt.cpp:62-75
  PrimeSet ps;
  ps.word = WordSize::w64;
  ps.two_n = 8;
  ps.primes = {17};
  ps.roots = {find_root_of_unity(17, 8)};
  ps.pair_one = {shoup_precompute(1, 17, WordSize::w64)};
  ps.pair_beta = {shoup_precompute((~uint64_t{0} % 17 + 1) % 17, 17, WordSize::w64)};
  ps.pair_beta2 = {shoup_precompute(
      mulmod_u64(ps.pair_beta[0].value, ps.pair_beta[0].value, 17), 17, WordSize::w64)};
  ps.product = bigint_from_u64(17, WordSize::w64);
  return ps;
}

struct Pipeline {  // test_polymul.cpp:45-67
  PrimeSet ps;
  CrtTables crt;
  NttTables ntt;
  IcrtTables icrt;
  PmContext ctx;
  Pipeline(int log_n, int log_q) {
    const WordSize w = WordSize::w64;
    int np = region1_prime_count(log_q, log_n, w);
    ps = generate_primes(np, log_n, w);
    while (bigint_cmp(ps.product, bigint_pow2(2 * log_q + log_n + 1, w)) < 0)
      ps = generate_primes(++np, log_n, w);
    crt = make_crt_tables(ps, log_q);
    ntt = make_ntt_tables(ps, log_n);
    icrt = make_icrt_tables(ps, bigint_pow2(log_q, w), w);
    ctx.ps = &ps;
    ctx.crt = &crt;
    ctx.ntt = &ntt;
    ctx.icrt = &icrt;
  }
};

void ntt_cases(bool quick) {
  run_case("word: Shoup known answer and exhaustive p=17 (SPEC.md:62, test_arith.cpp)", [] {
    const ShoupPair sp = shoup_precompute(3, 17, WordSize::w64);
    CHECK(shoup_modmul(5, sp, 17, WordSize::w64) == 15);
    for (uint64_t y = 0; y < 17; ++y) {
      const ShoupPair s = shoup_precompute(y, 17, WordSize::w64);
      for (uint64_t x = 0; x < 17; ++x) {
        CHECK(shoup_modmul(x, s, 17, WordSize::w64) == x * y % 17);
        CHECK(reduce_4p(shoup_modmul_approx(x, s, 17, WordSize::w64), 17) == x * y % 17);
        CHECK(shoup_modmul_lazy_t<64>(x, s, 17) < 34);
      }
    }
  });
  run_case("ntt: n=4 p=17 round trips and monomial products (test_ntt.cpp:60-101)", [quick] {
    const PrimeSet ps = p17_set();
    const NttTables t = make_ntt_tables(ps, 2);
    // [1,0,0,0] -> [1,1,1,1]
    RnsMatrix e = make_rns(1, 4, Layout::prime_major);
    e.at(0, 0) = 1;
    ntt_forward(e, ps, t);
    CHECK((e.data == std::vector<uint64_t>{1, 1, 1, 1}));
    const uint64_t total = 17ull * 17 * 17 * 17;
    for (uint64_t v = 0; v < total; v += quick ? 97 : 1) {
      RnsMatrix m = make_rns(1, 4, Layout::prime_major);
      uint64_t x = v;
      for (int i = 0; i < 4; ++i) m.at(0, i) = x % 17, x /= 17;
      RnsMatrix f = m;
      ntt_forward(f, ps, t);
      ntt_inverse(f, ps, t);
      CHECK(f.data == m.data);
    }
    for (int i = 0; i < 4; ++i)
      for (int j = 0; j < 4; ++j) {
        RnsMatrix a = make_rns(1, 4, Layout::prime_major), b = make_rns(1, 4, Layout::prime_major);
        a.at(0, i) = 3;
        b.at(0, j) = 5;
        RnsMatrix fa = a, fb = b, fr;
        ntt_forward(fa, ps, t);
        ntt_forward(fb, ps, t);
        rns_pointwise_mul(fr, fa, fb, ps);
        ntt_inverse(fr, ps, t);
        CHECK(fr.data == negacyclic_mod_p(a.data, b.data, 17));
      }
  });
  run_case("ntt: convolution across sizes and radices (test_ntt.cpp:104-117)", [] {
    Rng rng(55);
    for (int log_n : {3, 4, 6, 9, 12}) {
      const PrimeSet ps = generate_primes(3, log_n, WordSize::w64);
      const NttTables t = make_ntt_tables(ps, log_n);
      const int n = 1 << log_n;
      for (int radix_log : {1, 2, 4, 5}) {
        NttOptions opt;
        opt.radix_log = radix_log;
        const RnsMatrix a = random_matrix(ps, n, rng), b = random_matrix(ps, n, rng);
        RnsMatrix fa = a, fb = b, fr;
        ntt_forward(fa, ps, t, opt);
        ntt_forward(fb, ps, t, opt);
        rns_pointwise_mul(fr, fa, fb, ps);
        ntt_inverse(fr, ps, t, opt);
        for (int j = 0; j < 3; ++j) {
          std::vector<uint64_t> aj(a.data.begin() + j * n, a.data.begin() + (j + 1) * n);
          std::vector<uint64_t> bj(b.data.begin() + j * n, b.data.begin() + (j + 1) * n);
          std::vector<uint64_t> got(fr.data.begin() + j * n, fr.data.begin() + (j + 1) * n);
          if (log_n <= 9) CHECK(got == negacyclic_mod_p(aj, bj, ps.primes[j]));
        }
        RnsMatrix back = fa;
        ntt_inverse(back, ps, t, opt);
        CHECK(back.data == a.data);
      }
    }
  });
  run_case("ntt: radix / lazy / approx options give identical transforms (test_ntt.cpp:119-165)",
           [] {
             Rng rng(66);
             for (int log_n : {6, 10, 16}) {
               const PrimeSet ps = generate_primes(4, log_n, WordSize::w64);
               const NttTables t = make_ntt_tables(ps, log_n);
               const RnsMatrix a = random_matrix(ps, 1 << log_n, rng);
               RnsMatrix ref = a;
               ntt_forward(ref, ps, t);
               for (int radix_log : {2, 3, 4, 5})
                 for (bool lazy : {false, true}) {
                   NttOptions opt;
                   opt.radix_log = radix_log;
                   opt.lazy = opt.approx = lazy;
                   RnsMatrix f = a;
                   ntt_forward(f, ps, t, opt);
                   CHECK(f.data == ref.data);
                   ntt_inverse(f, ps, t, opt);
                   CHECK(f.data == a.data);
                 }
             }
             NttOptions bad;
             bad.radix_log = 6;
             const PrimeSet ps = generate_primes(1, 4, WordSize::w64);
             const NttTables t = make_ntt_tables(ps, 4);
             RnsMatrix m = make_rns(1, 16, Layout::prime_major);
             CHECK(throws<std::invalid_argument>([&] { ntt_forward(m, ps, t, bad); }));
             RnsMatrix cm = make_rns(1, 16, Layout::coeff_major);
             CHECK(throws<std::invalid_argument>([&] { ntt_forward(cm, ps, t); }));
           });
  run_case("ntt: memory passes and operation counters (test_ntt.cpp:167-194)", [] {
    CHECK(ntt_memory_passes(16, 1) == 16);
    CHECK(ntt_memory_passes(16, 2) == 8);
    CHECK(ntt_memory_passes(16, 4) == 4);
    CHECK(ntt_memory_passes(16, 5) == 4);
    CHECK(ntt_memory_passes(12, 5) == 3);
    const int log_n = 8, n = 256, np = 3;
    const PrimeSet ps = generate_primes(np, log_n, WordSize::w64);
    const NttTables t = make_ntt_tables(ps, log_n);
    Rng rng(88);
    RnsMatrix a = random_matrix(ps, n, rng);
    StageCounters cnt, cnt2;
    ntt_forward(a, ps, t, {}, nullptr, &cnt);
    CHECK(cnt[Stage::ntt].modmul == uint64_t(np) * n / 2 * log_n);
    CHECK(cnt[Stage::ntt].addsub == uint64_t(np) * n * log_n);
    ntt_inverse(a, ps, t, {}, nullptr, &cnt2);
    CHECK(cnt2[Stage::intt].modmul == uint64_t(np) * (n / 2 * log_n + n));
    CHECK(cnt2[Stage::intt].addsub == uint64_t(np) * n * log_n);
  });
}

void rns_cases() {
  run_case("rns: forward CRT residues, both layouts and strategies (test_rns.cpp:21-45)", [] {
    Rng rng(21);
    const int log_n = 6, n = 64, log_q = 150, np = 7;
    const PrimeSet ps = generate_primes(np, log_n, WordSize::w64);
    const CrtTables ct = make_crt_tables(ps, log_q);
    const BigPoly a = random_poly(n, log_q, rng);
    for (AccumKind kind : {AccumKind::three_word_adc, AccumKind::periodic_mod}) {
      AccumStrategy strat;
      strat.kind = kind;
      strat.period = kind == AccumKind::periodic_mod ? max_valid_period(ps) : 0;
      for (Layout layout : {Layout::prime_major, Layout::coeff_major}) {
        const RnsMatrix m = crt_forward(a, ps, ct, strat, layout);
        CHECK(m.layout == layout);
        for (int j = 0; j < np; ++j)
          for (int i = 0; i < n; ++i)
            CHECK(m.at(j, i) == bigint_mod_word(poly_get(a, i), ps.primes[j], WordSize::w64));
      }
    }
  });
  run_case("rns: accumulation strategy validity (test_rns.cpp:47-69)", [] {
    const PrimeSet ps64 = generate_primes(3, 8, WordSize::w64);
    const PrimeSet ps32 = generate_primes(3, 8, WordSize::w32);
    AccumStrategy s;
    s.kind = AccumKind::periodic_mod;
    s.period = 0;
    CHECK(!accum_strategy_valid(s, ps64));
    s.period = max_valid_period(ps64);
    CHECK(s.period >= 1);
    CHECK(accum_strategy_valid(s, ps64));
    s.period += 1;
    CHECK(!accum_strategy_valid(s, ps64));
    CHECK(max_valid_period(ps32) >= 2);
    const CrtTables ct = make_crt_tables(ps64, 100);
    Rng rng(1);
    const BigPoly a = random_poly(16, 100, rng);
    CHECK(throws<std::invalid_argument>([&] { crt_forward(a, ps64, ct, s, Layout::prime_major); }));
  });
  run_case("rns: CRT then iCRT is the identity, both variants (test_rns.cpp:71-91)", [] {
    Rng rng(33);
    for (int log_n : {5, 10}) {
      const int n = 1 << log_n, log_q = 140;
      const int np = region1_prime_count(log_q, log_n, WordSize::w64);
      const PrimeSet ps = generate_primes(np, log_n, WordSize::w64);
      const CrtTables ct = make_crt_tables(ps, log_q);
      const IcrtTables it = make_icrt_tables(ps, bigint_pow2(log_q, WordSize::w64), WordSize::w64);
      for (int t = 0; t < 5; ++t) {
        const BigPoly a = random_poly(n, log_q, rng);
        const RnsMatrix m = crt_forward(a, ps, ct, AccumStrategy{}, Layout::prime_major);
        const BigPoly b1 = icrt_naive(m, ps, it), b2 = icrt_reordered(m, ps, it);
        CHECK(poly_equal(a, b1));
        CHECK(b1.data == b2.data);
      }
    }
  });
  run_case("rns: iCRT near the product bound and negatives (test_rns.cpp:93-133)", [] {
    const WordSize w = WordSize::w64;
    const int np = 4, log_q = 100, n = 8;
    const PrimeSet ps = generate_primes(np, 6, w);
    const IcrtTables it = make_icrt_tables(ps, bigint_pow2(log_q, w), w);
    const BigInt P = ps.product, half = bigint_shr(P, 1, w), q = bigint_pow2(log_q, w);
    Rng rng(9);
    RnsMatrix m = make_rns(np, n, Layout::prime_major);
    std::vector<BigInt> vals(n);
    for (int i = 0; i < n; ++i) {
      vals[i] = bigint_from_u64(rng.next(), w);
      if (i % 2) {  // P - small: a centred negative
        BigInt d;
        bigint_sub(d, P, bigint_from_u64(rng.next(), w), w);
        vals[i] = d;
      }
      for (int j = 0; j < np; ++j) m.at(j, i) = bigint_mod_word(vals[i], ps.primes[j], w);
    }
    const BigPoly out = icrt_naive(m, ps, it), out2 = icrt_reordered(m, ps, it);
    CHECK(out.data == out2.data);
    for (int i = 0; i < n; ++i) {
      BigInt want;
      if (bigint_cmp(vals[i], half) > 0) {  // v - P mod q = q - ((P - v) mod q)
        BigInt d;
        bigint_sub(d, P, vals[i], w);
        const BigInt dm = bigint_mod(d, q, w);
        if (bigint_is_zero(dm))
          want = {};
        else
          bigint_sub(want, q, dm, w);
      } else {
        want = bigint_mod(vals[i], q, w);
      }
      bigint_trim(want);
      BigInt got = poly_get(out, i);
      bigint_trim(got);
      CHECK(bigint_cmp(got, want) == 0);
    }
  });
  run_case("rns: pointwise products and transpose (test_rns.cpp:135-167)", [] {
    Rng rng(44);
    const int np = 5, n = 64;
    const PrimeSet ps = generate_primes(np, 6, WordSize::w64);
    const RnsMatrix a = random_matrix(ps, n, rng), b = random_matrix(ps, n, rng);
    RnsMatrix r = make_rns(np, n, Layout::prime_major);
    rns_pointwise_mul(r, a, b, ps);
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < n; ++i) CHECK(r.at(j, i) == mulmod_u64(a.at(j, i), b.at(j, i), ps.primes[j]));
    RnsMatrix ta = a, tb = b, tr;
    rns_transpose(ta);
    rns_transpose(tb);
    rns_pointwise_mul(tr, ta, tb, ps);
    CHECK(tr.layout == Layout::coeff_major);
    for (int j = 0; j < np; ++j)
      for (int i = 0; i < n; ++i) CHECK(tr.at(j, i) == r.at(j, i));
    RnsMatrix m = make_rns(3, 4, Layout::prime_major);
    uint64_t v = 0;
    for (auto& x : m.data) x = v++;
    RnsMatrix t = m;
    rns_transpose(t);
    CHECK(t.layout == Layout::coeff_major);
    for (int j = 0; j < 3; ++j)
      for (int i = 0; i < 4; ++i) CHECK(t.at(j, i) == m.at(j, i));
    rns_transpose(t);
    CHECK(t.data == m.data);
  });
  run_case("rns: operation counters (test_rns.cpp:169-206)", [] {
    const int log_n = 5, n = 32, log_q = 140;
    const WordSize w = WordSize::w64;
    const int np = region1_prime_count(log_q, log_n, w);
    const PrimeSet ps = generate_primes(np, log_n, w);
    const CrtTables ct = make_crt_tables(ps, log_q);
    const IcrtTables it = make_icrt_tables(ps, bigint_pow2(log_q, w), w);
    Rng rng(2);
    const BigPoly a = random_poly(n, log_q, rng);
    StageCounters cnt, cnt2, cnt4;
    const RnsMatrix m = crt_forward(a, ps, ct, AccumStrategy{}, Layout::prime_major, nullptr, &cnt);
    const uint64_t cells = uint64_t(n) * np;
    CHECK(cnt[Stage::crt].mul == cells * ct.q_limbs);
    CHECK(cnt[Stage::crt].adc == cells * ct.q_limbs);
    CHECK(cnt[Stage::crt].modmul == cells);
    icrt_naive(m, ps, it, nullptr, &cnt2);
    CHECK(cnt2[Stage::icrt].mul == cells * it.p_limbs);
    CHECK(cnt2[Stage::icrt].modmul == cells);
    AccumStrategy per;
    per.kind = AccumKind::periodic_mod;
    per.period = max_valid_period(ps);
    crt_forward(a, ps, ct, per, Layout::prime_major, nullptr, &cnt4);
    CHECK(cnt4[Stage::crt].modmul == cells * ((ct.q_limbs + per.period - 1) / per.period));
  });
  run_case("rns: 32-bit words are rejected by the GPU path", [] {
    const PrimeSet ps = generate_primes(3, 6, WordSize::w32);
    const RnsMatrix a = make_rns(3, 64, Layout::prime_major);
    RnsMatrix r;
    CHECK(throws<std::invalid_argument>([&] { rns_pointwise_mul(r, a, a, ps); }));
  });
}

void polymul_cases() {
  run_case("polymul: pipeline = exact product = schoolbook (test_polymul.cpp:71-89)", [] {
    Rng rng(101);
    for (int log_n : {3, 5, 7}) {
      const int n = 1 << log_n, log_q = 120;
      Pipeline pl(log_n, log_q);
      for (int t = 0; t < 3; ++t) {
        const BigPoly a = random_poly(n, log_q, rng), b = random_poly(n, log_q, rng);
        const BigPoly want = exact_negacyclic(a, b);
        CHECK(poly_equal(poly_mul(a, b, pl.ctx), want));
        CHECK(poly_equal(schoolbook_negacyclic(a, b, bigint_pow2(log_q, WordSize::w64),
                                               WordSize::w64),
                         want));
      }
    }
  });
  run_case("polymul: options yield the identical product (test_polymul.cpp:91-117)", [] {
    Rng rng(202);
    const int log_n = 6, n = 64, log_q = 150;
    Pipeline pl(log_n, log_q);
    const BigPoly a = random_poly(n, log_q, rng), b = random_poly(n, log_q, rng);
    const BigPoly ref = poly_mul(a, b, pl.ctx);
    CHECK(poly_equal(ref, exact_negacyclic(a, b)));
    for (int radix_log : {1, 2, 4, 5})
      for (bool reord : {false, true})
        for (bool lazy : {false, true}) {
          Pipeline v(log_n, log_q);
          v.ctx.ntt_opt.radix_log = radix_log;
          v.ctx.ntt_opt.lazy = v.ctx.ntt_opt.approx = lazy;
          v.ctx.icrt_loop_reordered = reord;
          CHECK(poly_equal(poly_mul(a, b, v.ctx), ref));
        }
    Pipeline v(log_n, log_q);
    v.ctx.strategy.kind = AccumKind::periodic_mod;
    v.ctx.strategy.period = max_valid_period(v.ps);
    CHECK(poly_equal(poly_mul(a, b, v.ctx), ref));
  });
  run_case("polymul: prepared operands reused; paper-size ring (test_polymul.cpp:119-134)", [] {
    Rng rng(303);
    const int log_n = 4, n = 16, log_q = 100;
    Pipeline pl(log_n, log_q);
    const BigPoly a = random_poly(n, log_q, rng), b = random_poly(n, log_q, rng),
                  c = random_poly(n, log_q, rng);
    const RnsForm fa = pm_prepare(a, pl.ctx), fb = pm_prepare(b, pl.ctx), fc = pm_prepare(c, pl.ctx);
    CHECK(poly_equal(pm_finish(pm_pointwise(fa, fb, pl.ctx), pl.ctx), exact_negacyclic(a, b)));
    CHECK(poly_equal(pm_finish(pm_pointwise(fa, fc, pl.ctx), pl.ctx), exact_negacyclic(a, c)));
    // a large ring through the tiled kernels: (a b) c = a (b c)
    Pipeline big(14, 600);
    const int N = 1 << 14;
    const BigPoly x = random_poly(N, 600, rng), y = random_poly(N, 600, rng),
                  z = random_poly(N, 600, rng);
    CHECK(poly_equal(poly_mul(poly_mul(x, y, big.ctx), z, big.ctx),
                     poly_mul(x, poly_mul(y, z, big.ctx), big.ctx)));
  });
  run_case("polymul: schoolbook cap and pipeline counters (test_polymul.cpp:136-164)", [] {
    BigPoly big = make_poly(512, 60, WordSize::w64);
    CHECK(throws<std::invalid_argument>(
        [&] { schoolbook_negacyclic(big, big, bigint_pow2(60, WordSize::w64), WordSize::w64); }));
    Rng rng(404);
    const int log_n = 5, n = 32, log_q = 120;
    Pipeline pl(log_n, log_q);
    StageCounters cnt;
    StageTimers tim;
    pl.ctx.counters = &cnt;
    pl.ctx.timers = &tim;
    poly_mul(random_poly(n, log_q, rng), random_poly(n, log_q, rng), pl.ctx);
    const int np = static_cast<int>(pl.ps.primes.size());
    const uint64_t cells = uint64_t(n) * np;
    CHECK(cnt[Stage::crt].mul == 2 * cells * pl.crt.q_limbs);
    CHECK(cnt[Stage::ntt].modmul == 2 * uint64_t(np) * n / 2 * log_n);
    CHECK(cnt[Stage::intt].modmul == uint64_t(np) * (n / 2 * log_n + n));
    CHECK(cnt[Stage::icrt].mul == cells * pl.icrt.p_limbs);
    CHECK(cnt[Stage::icrt].modmul == 2 * cells);
    CHECK(tim.total() > 0);
  });
}

}  // namespace

int main(int argc, char** argv) {
  const bool quick = argc > 1 && std::strcmp(argv[1], "--quick") == 0;
  ntt_cases(quick);
  rns_cases();
  polymul_cases();
  std::printf("checks %d failures %d\n", g_checks, g_failures);
  return g_failures ? 1 : 0;
}
