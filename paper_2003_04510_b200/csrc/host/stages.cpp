// The reference's lower-level stage API (include/hemul/rns.hpp, ntt.hpp,
// polymul.hpp) on the GPU.
//
// crt_forward / rns_pointwise_mul / icrt_* / ntt_forward / ntt_inverse call
// the explicit-prime-set C-ABI (hemul_gpu_rns_*, include/hemul_gpu.h), which
// runs the same CRT / pointwise / NTT / iCRT kernels as the stage entry
// points on tables built from the caller's PrimeSet (csrc/level_tables.cpp
// build_explicit_region) and uploaded once per (prime set, ring degree,
// widths). Operation counts and stage timers follow the reference's
// bookkeeping exactly (rns.cpp:331-415, ntt.cpp:153-197, polymul.cpp:7-43).
// Without a usable GPU every computing call throws (no CPU fallback).
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>

#include "hemul/polymul.hpp"
#include "hemul_gpu.h"

namespace hemul {

namespace {

// One process-wide device context for the stage functions (they are free
// functions in the reference); calls are serialised.
struct StageDevice {
  std::mutex mu;
  hemul_gpu_ctx* ctx = nullptr;
  struct Entry {
    std::vector<uint64_t> primes, roots;  // roots empty: no NTT tables
    int log_n, in_bits, target_bits;
    hemul_gpu_rns* h;
  };
  std::list<Entry> cache;  // most recent first
  static constexpr size_t kCapacity = 16;

  ~StageDevice() {
    for (auto& e : cache) hemul_gpu_rns_destroy(e.h);
    if (ctx) hemul_gpu_destroy(ctx);
  }

  hemul_gpu_ctx* get() {
    if (!ctx) {
      const char* env = std::getenv("HEMUL_DEVICE");
      // the context parameters are irrelevant here: only its device and
      // stream are used (the prime-set objects carry their own ring degree)
      if (hemul_gpu_create(env ? std::atoi(env) : 0, 30, 2, 12, &ctx) != HEMUL_OK) {
        ctx = nullptr;
        throw std::runtime_error("hemul_gpu_create failed: no usable CUDA device");
      }
    }
    return ctx;
  }

  [[noreturn]] void fail(hemul_status st) {
    const std::string msg = ctx ? hemul_gpu_last_error(ctx) : "no GPU context";
    if (st == HEMUL_E_ARG) throw std::invalid_argument(msg);
    throw std::runtime_error("hemul_gpu: " + msg);
  }

  void check(hemul_status st) {
    if (st != HEMUL_OK) fail(st);
  }

  // ntt = false: CRT / pointwise / iCRT tables only (the set's roots may be
  // for another ring degree, e.g. test_rns.cpp:93-133)
  hemul_gpu_rns* tables(const PrimeSet& ps, int log_n, int in_bits, int target_bits, bool ntt) {
    const std::vector<uint64_t> roots = ntt ? ps.roots : std::vector<uint64_t>{};
    for (auto it = cache.begin(); it != cache.end(); ++it)
      if (it->log_n == log_n && it->in_bits == in_bits && it->target_bits == target_bits &&
          it->primes == ps.primes && it->roots == roots) {
        cache.splice(cache.begin(), cache, it);
        return cache.front().h;
      }
    hemul_gpu_rns* h = nullptr;
    check(hemul_gpu_rns_create(get(), log_n, ps.primes.data(), ntt ? roots.data() : nullptr,
                               static_cast<int>(ps.primes.size()), in_bits, target_bits, &h));
    cache.push_front(Entry{ps.primes, roots, log_n, in_bits, target_bits, h});
    while (cache.size() > kCapacity) {
      hemul_gpu_rns_destroy(cache.back().h);
      cache.pop_back();
    }
    return h;
  }
};

StageDevice& device() {
  static StageDevice d;
  return d;
}

int log2_exact(int n) {
  if (n <= 0 || (n & (n - 1))) throw std::invalid_argument("ring degree must be a power of two");
  int l = 0;
  while ((1 << l) < n) ++l;
  return l;
}

void require_w64(WordSize w) {
  if (w != WordSize::w64)
    throw std::invalid_argument("the B200 stage kernels support 64-bit words only");
}

// ScopedStageTimer (counters.hpp:58-76) for the synchronous GPU calls
struct Timer {
  StageTimers* t;
  Stage s;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  ~Timer() {
    if (t) (*t)[s] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
};

}  // namespace

// ---- RnsMatrix (rns.cpp:292-311) -------------------------------------------

RnsMatrix make_rns(int np, int n, Layout layout) {
  RnsMatrix m;
  m.np = np;
  m.n = n;
  m.layout = layout;
  m.data.assign(static_cast<size_t>(np) * n, 0);
  return m;
}

void rns_transpose(RnsMatrix& m) {
  RnsMatrix t = make_rns(m.np, m.n, m.layout == Layout::prime_major ? Layout::coeff_major
                                                                    : Layout::prime_major);
  for (int j = 0; j < m.np; ++j)
    for (int i = 0; i < m.n; ++i) t.at(j, i) = m.at(j, i);
  m = std::move(t);
}

// ---- accumulation strategies (rns.cpp:34-41, 313-329) ------------------------

namespace {

bool period_ok(int period, uint64_t p, WordSize w) {
  using u128 = unsigned __int128;
  if (period < 1) return false;
  if (w == WordSize::w32) {
    const u128 beta = u128{1} << 32;
    return p + u128(period) * (beta - 1) * (p - 1) < beta * beta;
  }
  // p + period (2^64 - 1)(p - 1) must not exceed 2^128 - 1
  const u128 term = u128(~uint64_t{0}) * (p - 1);
  return term == 0 || u128(period) <= (~u128{0} - p) / term;
}

}  // namespace

bool accum_strategy_valid(const AccumStrategy& s, const PrimeSet& ps) {
  if (s.kind == AccumKind::three_word_adc) return true;
  for (uint64_t p : ps.primes)
    if (!period_ok(s.period, p, ps.word)) return false;
  return true;
}

int max_valid_period(const PrimeSet& ps) {
  int best = 0;
  for (int per = 1; per <= 64; ++per) {
    for (uint64_t p : ps.primes)
      if (!period_ok(per, p, ps.word)) return best;
    best = per;
  }
  return best;
}

// ---- CRT / pointwise / iCRT ------------------------------------------------

RnsMatrix crt_forward(const BigPoly& a, const PrimeSet& ps, const CrtTables& ct,
                      const AccumStrategy& strat, Layout out_layout, ThreadPool*,
                      StageCounters* cnt, StageTimers* tim) {
  if (strat.kind == AccumKind::periodic_mod && !accum_strategy_valid(strat, ps))
    throw std::invalid_argument("accumulation period too large for prime set");
  require_w64(a.word);
  Timer timer{tim, Stage::crt};
  const int log_n = log2_exact(a.n);
  const int ql = ct.q_limbs;
  // the kernel reads q_limbs limbs per coefficient (rns.cpp:47-58)
  std::vector<uint64_t> staged;
  const uint64_t* src = a.data.data();
  if (a.limbs != ql) {
    staged.assign(static_cast<size_t>(a.n) * ql, 0);
    const int keep = std::min(a.limbs, ql);
    for (int i = 0; i < a.n; ++i)
      std::memcpy(&staged[static_cast<size_t>(i) * ql], a.coeff(i), sizeof(uint64_t) * keep);
    src = staged.data();
  }
  RnsMatrix out = make_rns(ct.np, a.n, Layout::prime_major);
  {
    StageDevice& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    hemul_gpu_rns* h = d.tables(ps, log_n, 64 * ql, 0, false);
    d.check(hemul_gpu_rns_crt(d.get(), h, 1, src, out.data.data()));
  }
  if (cnt) {
    const uint64_t cells = static_cast<uint64_t>(a.n) * ct.np;
    auto& c = (*cnt)[Stage::crt];
    c.mul += cells * ql;
    c.adc += cells * ql;
    c.modmul += cells * (strat.kind == AccumKind::three_word_adc
                             ? 1
                             : (ql + strat.period - 1) / strat.period);
  }
  if (out_layout == Layout::coeff_major) rns_transpose(out);
  return out;
}

void rns_pointwise_mul(RnsMatrix& r, const RnsMatrix& a, const RnsMatrix& b, const PrimeSet& ps,
                       ThreadPool*, StageCounters* cnt, StageTimers* tim) {
  if (a.np != b.np || a.n != b.n || a.layout != b.layout)
    throw std::invalid_argument("pointwise operands differ in shape or layout");
  require_w64(ps.word);
  Timer timer{tim, Stage::icrt};  // booked like rns.cpp:362-371
  if (r.np != a.np || r.n != a.n) r = make_rns(a.np, a.n, a.layout);
  r.layout = a.layout;
  // elementwise: a coefficient-major pair is handled as its transposes
  const bool cm = a.layout == Layout::coeff_major;
  RnsMatrix ta, tb;
  const RnsMatrix* pa = &a;
  const RnsMatrix* pb = &b;
  if (cm) {
    ta = a;
    tb = b;
    rns_transpose(ta);
    rns_transpose(tb);
    pa = &ta;
    pb = &tb;
  }
  RnsMatrix out = make_rns(a.np, a.n, Layout::prime_major);
  {
    StageDevice& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    hemul_gpu_rns* h = d.tables(ps, log2_exact(a.n), 0, 0, false);
    d.check(hemul_gpu_rns_pointwise(d.get(), h, 1, pa->data.data(), pb->data.data(),
                                    out.data.data()));
  }
  if (cm) rns_transpose(out);
  r = std::move(out);
  if (cnt) (*cnt)[Stage::icrt].modmul += static_cast<uint64_t>(a.n) * a.np;
}

namespace {

BigPoly icrt_gpu(const RnsMatrix& m, const PrimeSet& ps, const IcrtTables& t, StageCounters* cnt,
                 StageTimers* tim) {
  require_w64(ps.word);
  if (!t.target_pow2 || t.target_log2 <= 0)
    throw std::invalid_argument("the B200 iCRT reconstructs modulo powers of two only");
  Timer timer{tim, Stage::icrt};
  RnsMatrix pm;
  const RnsMatrix* src = &m;
  if (m.layout != Layout::prime_major) {
    pm = m;
    rns_transpose(pm);
    src = &pm;
  }
  BigPoly r = make_poly(m.n, t.target_log2, WordSize::w64);
  {
    StageDevice& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    hemul_gpu_rns* h = d.tables(ps, log2_exact(m.n), 0, t.target_log2, false);
    d.check(hemul_gpu_rns_icrt(d.get(), h, 1, src->data.data(), r.data.data()));
  }
  if (cnt) {
    const uint64_t cells = static_cast<uint64_t>(m.n) * t.np;
    auto& c = (*cnt)[Stage::icrt];
    c.modmul += cells;
    c.mul += cells * t.p_limbs;
    c.adc += cells * t.p_limbs;
  }
  return r;
}

}  // namespace

// Both loop orders are one GPU kernel: the reference proves them
// bit-identical (rns.hpp:74-78).
BigPoly icrt_naive(const RnsMatrix& m, const PrimeSet& ps, const IcrtTables& t, ThreadPool*,
                   StageCounters* cnt, StageTimers* tim) {
  return icrt_gpu(m, ps, t, cnt, tim);
}

BigPoly icrt_reordered(const RnsMatrix& m, const PrimeSet& ps, const IcrtTables& t, ThreadPool*,
                       StageCounters* cnt, StageTimers* tim) {
  return icrt_gpu(m, ps, t, cnt, tim);
}

// ---- NTT (ntt.cpp:139-197) -----------------------------------------------------

int ntt_memory_passes(int log_n, int radix_log) { return (log_n + radix_log - 1) / radix_log; }

namespace {

void ntt_gpu(RnsMatrix& m, const PrimeSet& ps, const NttTables& t, const NttOptions& opt,
             bool inverse, StageCounters* cnt, StageTimers* tim) {
  if (m.layout != Layout::prime_major)
    throw std::invalid_argument("transforms expect prime-major layout");
  if (m.n != t.n) throw std::invalid_argument("size mismatch with tables");
  if (opt.radix_log < 1 || opt.radix_log > 5)
    throw std::invalid_argument("radix_log must be in [1, 5]");
  require_w64(ps.word);
  Timer timer{tim, inverse ? Stage::intt : Stage::ntt};
  {
    StageDevice& d = device();
    std::lock_guard<std::mutex> lock(d.mu);
    hemul_gpu_rns* h = d.tables(ps, t.log_n, 0, 0, true);
    d.check(hemul_gpu_rns_ntt(d.get(), h, m.data.data(), static_cast<size_t>(m.np),
                              inverse ? 1 : 0));
  }
  if (cnt) {
    const uint64_t bf = static_cast<uint64_t>(m.np) * (m.n / 2) * t.log_n;
    auto& c = (*cnt)[inverse ? Stage::intt : Stage::ntt];
    c.modmul += bf + (inverse ? static_cast<uint64_t>(m.np) * m.n : 0);
    c.addsub += 2 * bf;
  }
}

}  // namespace

void ntt_forward(RnsMatrix& m, const PrimeSet& ps, const NttTables& t, const NttOptions& opt,
                 ThreadPool*, StageCounters* cnt, StageTimers* tim) {
  ntt_gpu(m, ps, t, opt, false, cnt, tim);
}

void ntt_inverse(RnsMatrix& m, const PrimeSet& ps, const NttTables& t, const NttOptions& opt,
                 ThreadPool*, StageCounters* cnt, StageTimers* tim) {
  ntt_gpu(m, ps, t, opt, true, cnt, tim);
}

// ---- the product pipeline (polymul.cpp:7-43) ---------------------------------

RnsForm pm_prepare(const BigPoly& a, const PmContext& ctx) {
  RnsForm f;
  // the GPU CRT writes prime-major rows directly: the reference's
  // coefficient-major result and transposition pass (polymul.cpp:11-16) are
  // not needed; the (empty) extra-stage time is still booked
  f.m = crt_forward(a, *ctx.ps, *ctx.crt, ctx.strategy, Layout::prime_major, ctx.pool,
                    ctx.counters, ctx.timers);
  { Timer t{ctx.timers, Stage::extra}; }
  ntt_forward(f.m, *ctx.ps, *ctx.ntt, ctx.ntt_opt, ctx.pool, ctx.counters, ctx.timers);
  return f;
}

RnsMatrix pm_pointwise(const RnsForm& a, const RnsForm& b, const PmContext& ctx) {
  RnsMatrix r;
  rns_pointwise_mul(r, a.m, b.m, *ctx.ps, ctx.pool, ctx.counters, ctx.timers);
  return r;
}

BigPoly pm_finish(RnsMatrix prod, const PmContext& ctx) {
  ntt_inverse(prod, *ctx.ps, *ctx.ntt, ctx.ntt_opt, ctx.pool, ctx.counters, ctx.timers);
  return ctx.icrt_loop_reordered
             ? icrt_reordered(prod, *ctx.ps, *ctx.icrt, ctx.pool, ctx.counters, ctx.timers)
             : icrt_naive(prod, *ctx.ps, *ctx.icrt, ctx.pool, ctx.counters, ctx.timers);
}

BigPoly poly_mul(const BigPoly& a, const BigPoly& b, const PmContext& ctx) {
  const RnsForm fa = pm_prepare(a, ctx);
  const RnsForm fb = pm_prepare(b, ctx);
  return pm_finish(pm_pointwise(fa, fb, ctx), ctx);
}

// The reference's quadratic cross-check (polymul.cpp:45-88), host code: it is
// the independent check of the GPU pipeline above, not a path of it.
BigPoly schoolbook_negacyclic(const BigPoly& a, const BigPoly& b, const BigInt& modulus,
                              WordSize w) {
  if (a.n > 256) throw std::invalid_argument("schoolbook reference capped at n = 256");
  const int n = a.n;
  std::vector<BigInt> plus(static_cast<size_t>(n)), minus(static_cast<size_t>(n));
  auto accumulate = [&](BigInt& acc, const BigInt& v) {
    BigInt s;
    const uint64_t carry = bigint_add(s, acc, v, w);
    if (carry) s.push_back(carry);
    acc = std::move(s);
  };
  for (int i = 0; i < n; ++i) {
    const BigInt ai = poly_get(a, i);
    if (bigint_is_zero(ai)) continue;
    for (int j = 0; j < n; ++j) {
      const BigInt bj = poly_get(b, j);
      if (bigint_is_zero(bj)) continue;
      // X^(i+j) = -X^(i+j-n) past the ring degree
      accumulate(i + j < n ? plus[i + j] : minus[i + j - n], bigint_mul(ai, bj, w));
    }
  }
  int bits = bigint_bit_length(modulus, w);
  if (bits > 0 && bigint_cmp(modulus, bigint_pow2(bits - 1, w)) == 0) --bits;  // 2^k: k bits
  BigPoly r = make_poly(n, bits ? bits : 1, w);
  for (int i = 0; i < n; ++i) {
    BigInt u = bigint_mod(plus[i], modulus, w);
    const BigInt v = bigint_mod(minus[i], modulus, w);
    if (bigint_cmp(u, v) < 0) accumulate(u, modulus);
    BigInt diff;
    bigint_sub(diff, u, v, w);
    poly_set(r, i, diff);
  }
  return r;
}

}  // namespace hemul
