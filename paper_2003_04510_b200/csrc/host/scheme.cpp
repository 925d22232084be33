// hemul::Scheme of the drop-in API (include/hemul/heaan.hpp).
//
// Host side: CKKS slot encoding, key generation, encryption, decryption and
// the ternary products they use, reproducing proj/core/src/heaan.cpp:173-326
// arithmetic and RNG draw order exactly (the bench protocol's digests depend
// on it). GPU side: he_mul / rescale / warm_level call the C-ABI
// (include/hemul_gpu.h) with the BigPoly buffers as they are.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <numbers>
#include <stdexcept>
#include <string>

#include "hemul/heaan.hpp"
#include "hemul/io.hpp"
#include "hemul_gpu.h"

namespace hemul {

namespace {

// a[idx] += v for a small signed v, mod 2^log_q (heaan.cpp:53-71)
void add_signed(BigPoly& a, int idx, int64_t v) {
  if (v == 0) return;
  const WordSize w = a.word;
  BigInt c = poly_get(a, idx);
  if (v > 0) {
    bigint_add_word(c, static_cast<uint64_t>(v), w);
  } else {
    const BigInt m = bigint_from_u64(static_cast<uint64_t>(-v), w);
    if (bigint_cmp(c, m) >= 0) {
      bigint_sub(c, c, m, w);
    } else {
      BigInt q = bigint_pow2(a.log_q, w);
      bigint_sub(q, q, m, w);
      bigint_add(c, c, q, w);  // the wrap is masked off by poly_set
    }
  }
  poly_set(a, idx, c);
}

void add_error(BigPoly& a, const std::vector<int>& e) {
  for (int i = 0; i < a.n; ++i) add_signed(a, i, e[static_cast<size_t>(i)]);
}

BigPoly random_poly(Rng& rng, int n, int log_q, WordSize w) {
  BigPoly r = make_poly(n, log_q, w);
  for (int i = 0; i < n; ++i) poly_set(r, i, rng.uniform_bits(log_q, w));
  return r;
}

double limbs_to_double(const BigInt& v, WordSize w) {
  double r = 0;
  for (size_t k = v.size(); k-- > 0;) r = std::ldexp(r, log_beta(w)) + static_cast<double>(v[k]);
  return r;
}

// coefficient i of a in (-q/2, q/2] as a double (heaan.cpp:91-100)
double centered(const BigPoly& a, int i) {
  const BigInt c = poly_get(a, i);
  if (bigint_bit(c, a.log_q - 1, a.word)) {
    BigInt q = bigint_pow2(a.log_q, a.word);
    bigint_sub(q, q, c, a.word);
    return -limbs_to_double(q, a.word);
  }
  return limbs_to_double(c, a.word);
}

bool is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

[[noreturn]] void throw_status(hemul_gpu_ctx* g, hemul_status st) {
  const std::string msg = g ? hemul_gpu_last_error(g) : "no GPU context";
  switch (st) {
    case HEMUL_E_IO:
      throw IoError(msg);
    case HEMUL_E_MODULUS_MISMATCH:
    case HEMUL_E_ARG:
      throw std::invalid_argument(msg);
    case HEMUL_E_DEPTH:
      throw std::runtime_error(msg);
    default:
      throw std::runtime_error("hemul_gpu: " + msg);
  }
}

}  // namespace

Scheme::Scheme(const Params& params, ThreadPool* pool, int device)
    : params_(params), pool_(pool), device_(device) {
  if (device_ < 0) {
    const char* env = std::getenv("HEMUL_DEVICE");
    device_ = env ? std::atoi(env) : 0;
  }
}

Scheme::~Scheme() {
  if (ctx_) hemul_gpu_destroy(ctx_);
}

hemul_gpu_ctx* Scheme::gpu() const {
  if (!ctx_) {
    if (params_.word != WordSize::w64)
      throw std::invalid_argument("the B200 HE Mul path supports 64-bit words only");
    const hemul_status st =
        hemul_gpu_create(device_, params_.log_p, params_.depth, params_.log_n, &ctx_);
    if (st != HEMUL_OK) {
      ctx_ = nullptr;
      throw std::runtime_error("hemul_gpu_create failed (status " + std::to_string(st) +
                               "): no usable CUDA device");
    }
    hemul_gpu_enable_stage_timing(ctx_, 1);
  }
  return ctx_;
}

// ---- encoding (heaan.cpp:173-232) -------------------------------------------

Plaintext Scheme::encode(const Message& m) const {
  const int ns = static_cast<int>(m.slots.size());
  if (!is_pow2(ns) || 2 * ns > params_.n)
    throw std::invalid_argument("slot count must be a power of two <= N/2");
  const int two_ns = 2 * ns, four_ns = 4 * ns;
  const int gap = params_.n / two_ns;
  const double delta = std::ldexp(1.0, params_.log_delta);
  const double pi = std::numbers::pi;
  std::vector<int> rot(static_cast<size_t>(ns));  // 5^k mod 4 ns
  rot[0] = 1;
  for (int k = 1; k < ns; ++k) rot[k] = (rot[k - 1] * 5) % four_ns;
  Plaintext t;
  t.poly = make_poly(params_.n, params_.log_q_max, params_.word);
  t.log_q = params_.log_q_max;
  t.log_delta = params_.log_delta;
  t.n_slots = ns;
  for (int j = 0; j < two_ns; ++j) {
    double acc = 0;
    for (int k = 0; k < ns; ++k) {
      const int e = (four_ns - (static_cast<long long>(j) * rot[k]) % four_ns) % four_ns;
      const double ang = pi * e / (2.0 * ns);
      acc += m.slots[k].real() * std::cos(ang) - m.slots[k].imag() * std::sin(ang);
    }
    add_signed(t.poly, j * gap, std::llround(delta * acc / ns));
  }
  return t;
}

Message Scheme::decode(const Plaintext& t) const {
  const int ns = t.n_slots, n = params_.n, two_n = 2 * n;
  const double inv_delta = std::ldexp(1.0, -t.log_delta);
  const double pi = std::numbers::pi;
  std::vector<std::complex<double>> zeta(static_cast<size_t>(two_n));
  for (int e = 0; e < two_n; ++e) zeta[e] = {std::cos(pi * e / n), std::sin(pi * e / n)};
  std::vector<double> coeffs(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) coeffs[i] = centered(t.poly, i);
  std::vector<int> rot(static_cast<size_t>(ns));
  rot[0] = 1;
  for (int k = 1; k < ns; ++k) rot[k] = static_cast<int>((static_cast<long long>(rot[k - 1]) * 5) % two_n);
  Message m;
  m.slots.resize(static_cast<size_t>(ns));
  for (int k = 0; k < ns; ++k) {
    std::complex<double> z = 0;
    long long e = 0;
    for (int i = 0; i < n; ++i) {
      if (coeffs[i] != 0) z += coeffs[i] * zeta[static_cast<size_t>(e)];
      e += rot[k];
      if (e >= two_n) e -= two_n;
    }
    m.slots[k] = z * inv_delta;
  }
  return m;
}

// ---- ternary products and keys (heaan.cpp:234-315) ---------------------------

// On the GPU (hemul_gpu_mul_by_ternary: one thread per output coefficient
// over the limb-major polynomial, exact carries); the ternary vector and
// everything drawn from the RNG stay host-side.
BigPoly Scheme::mul_by_ternary(const BigPoly& a, const std::vector<int>& t) const {
  if (static_cast<int>(t.size()) != a.n) throw std::invalid_argument("ternary size mismatch");
  if (a.word != WordSize::w64 || a.n != params_.n)
    throw std::invalid_argument("mul_by_ternary: 64-bit words at the scheme's ring degree");
  hemul_gpu_ctx* g = gpu();
  BigPoly r = make_poly(a.n, a.log_q, a.word);
  static_assert(sizeof(int) == sizeof(int32_t), "int32 ternary vector");
  const hemul_status st = hemul_gpu_mul_by_ternary(g, a.log_q, 1, a.data.data(),
                                                   reinterpret_cast<const int32_t*>(t.data()),
                                                   r.data.data());
  if (st != HEMUL_OK) throw_status(g, st);
  return r;
}

KeySet Scheme::keygen(Rng& rng) const {
  const WordSize w = params_.word;
  const int n = params_.n, log_Q = params_.log_q_max;
  KeySet ks;
  ks.sk.s = rng.ternary_hwt(n, std::min(opts_.hamming_weight, n / 2));
  // pk = (a, -a s + e) mod Q
  ks.pk.ax = random_poly(rng, n, log_Q, w);
  poly_negate(ks.pk.bx, mul_by_ternary(ks.pk.ax, ks.sk.s));
  add_error(ks.pk.bx, rng.gaussian(n));
  // evk = (a', -a' s + e' + Q s^2) mod Q^2
  ks.evk.ax = random_poly(rng, n, 2 * log_Q, w);
  poly_negate(ks.evk.bx, mul_by_ternary(ks.evk.ax, ks.sk.s));
  add_error(ks.evk.bx, rng.gaussian(n));
  BigPoly s_poly = make_poly(n, 2 * log_Q, w);
  for (int i = 0; i < n; ++i) add_signed(s_poly, i, ks.sk.s[static_cast<size_t>(i)]);
  const BigPoly s2 = mul_by_ternary(s_poly, ks.sk.s);
  BigPoly qs2 = make_poly(n, 2 * log_Q, w);
  for (int i = 0; i < n; ++i) poly_set(qs2, i, bigint_shl(poly_get(s2, i), log_Q, w));
  poly_add(ks.evk.bx, ks.evk.bx, qs2);
  return ks;
}

Ciphertext Scheme::encrypt(const Plaintext& t, const PublicKey& pk, Rng& rng) const {
  if (t.log_q != params_.log_q_max)
    throw std::invalid_argument("plaintext must be at the fresh modulus");
  const int n = params_.n;
  const std::vector<int> u = rng.ternary_hwt(n, std::min(opts_.hamming_weight, n / 4));
  Ciphertext c;
  c.ax = mul_by_ternary(pk.ax, u);
  add_error(c.ax, rng.gaussian(n));
  c.bx = mul_by_ternary(pk.bx, u);
  add_error(c.bx, rng.gaussian(n));
  poly_add(c.bx, c.bx, t.poly);
  c.log_q = params_.log_q_max;
  c.n_slots = t.n_slots;
  return c;
}

Plaintext Scheme::decrypt(const Ciphertext& c, const SecretKey& sk) const {
  if (c.log_q < params_.log_p) throw std::runtime_error("modulus exhausted; cannot decrypt");
  Plaintext t;
  poly_add(t.poly, c.bx, mul_by_ternary(c.ax, sk.s));
  t.log_q = c.log_q;
  t.log_delta = params_.log_delta;
  t.n_slots = c.n_slots;
  return t;
}

Ciphertext Scheme::he_add(const Ciphertext& c1, const Ciphertext& c2) const {
  if (c1.log_q != c2.log_q) throw std::invalid_argument("ciphertext modulus mismatch");
  Ciphertext r;
  poly_add(r.ax, c1.ax, c2.ax);
  poly_add(r.bx, c1.bx, c2.bx);
  r.log_q = c1.log_q;
  r.n_slots = std::max(c1.n_slots, c2.n_slots);
  return r;
}

// ---- GPU entry points (heaan.cpp:119-171, 328-410) ---------------------------

void Scheme::warm_level(int log_q, const EvalKey* evk) {
  hemul_gpu_ctx* g = gpu();
  hemul_status st;
  if (evk) {
    st = hemul_gpu_set_evk(g, log_q, evk->ax.data.data(), evk->bx.data.data(),
                           reinterpret_cast<uintptr_t>(evk));
    evk_src_ = evk;
  } else {
    st = hemul_gpu_set_level(g, log_q);
  }
  if (st != HEMUL_OK) throw_status(g, st);
}

Ciphertext Scheme::rescale(const Ciphertext& c) const {
  if (c.log_q - params_.log_p < params_.log_p)
    throw std::runtime_error("modulus exhausted; cannot rescale");
  hemul_gpu_ctx* g = gpu();
  Ciphertext r;
  r.ax = make_poly(c.ax.n, c.log_q - params_.log_p, params_.word);
  r.bx = make_poly(c.bx.n, c.log_q - params_.log_p, params_.word);
  const hemul_status st = hemul_gpu_rescale(g, c.log_q, 1, c.ax.data.data(), c.bx.data.data(),
                                            r.ax.data.data(), r.bx.data.data());
  if (st != HEMUL_OK) throw_status(g, st);
  r.log_q = c.log_q - params_.log_p;
  r.n_slots = c.n_slots;
  return r;
}

Ciphertext Scheme::he_mul(const Ciphertext& c1, const Ciphertext& c2, const EvalKey& evk) {
  // the reference's checks, in order (heaan.cpp:341-345)
  if (c1.log_q != c2.log_q) throw std::invalid_argument("ciphertext modulus mismatch");
  const int log_q = c1.log_q;
  if (log_q - params_.log_p < params_.log_p)
    throw std::runtime_error("multiplicative depth exhausted");
  hemul_gpu_ctx* g = gpu();
  Ciphertext out;
  out.ax = make_poly(params_.n, log_q - params_.log_p, params_.word);
  out.bx = make_poly(params_.n, log_q - params_.log_p, params_.word);
  // evk identity = address, like the reference's level cache (heaan.cpp:152)
  const hemul_status st = hemul_gpu_he_mul(
      g, c1.log_q, c2.log_q, 1, c1.ax.data.data(), c1.bx.data.data(), c2.ax.data.data(),
      c2.bx.data.data(), evk.ax.data.data(), evk.bx.data.data(), reinterpret_cast<uintptr_t>(&evk),
      out.ax.data.data(), out.bx.data.data());
  if (st != HEMUL_OK) throw_status(g, st);
  evk_src_ = &evk;
  out.log_q = log_q - params_.log_p;
  out.n_slots = std::max(c1.n_slots, c2.n_slots);
  double ms[HEMUL_STAGE_COUNT] = {};
  if (hemul_gpu_stage_ms(g, ms) == HEMUL_OK)
    for (int s = 0; s < HEMUL_STAGE_COUNT; ++s) timers.seconds[s] += ms[s] * 1e-3;
  count_he_mul(log_q);
  return out;
}

// ---- device-resident ciphertexts ---------------------------------------------

DeviceCiphertext::DeviceCiphertext(hemul_gpu_ctx* ctx, hemul_gpu_ct* h, int q, int slots)
    : log_q(q), n_slots(slots), ctx_(ctx), h_(h) {}

DeviceCiphertext::~DeviceCiphertext() { hemul_gpu_ct_destroy(ctx_, h_); }

DeviceCiphertext::DeviceCiphertext(DeviceCiphertext&& o) noexcept
    : log_q(o.log_q), n_slots(o.n_slots), ctx_(o.ctx_), h_(o.h_) {
  o.h_ = nullptr;
}

DeviceCiphertext& DeviceCiphertext::operator=(DeviceCiphertext&& o) noexcept {
  if (this != &o) {
    hemul_gpu_ct_destroy(ctx_, h_);
    log_q = o.log_q;
    n_slots = o.n_slots;
    ctx_ = o.ctx_;
    h_ = o.h_;
    o.h_ = nullptr;
  }
  return *this;
}

DeviceCiphertext Scheme::upload(const Ciphertext& c) const {
  hemul_gpu_ctx* g = gpu();
  if (c.ax.log_q != c.log_q || c.bx.log_q != c.log_q || c.ax.n != params_.n)
    throw std::invalid_argument("ciphertext polynomials do not match its modulus");
  hemul_gpu_ct* h = nullptr;
  const hemul_status st =
      hemul_gpu_ct_create(g, c.log_q, 1, c.ax.data.data(), c.bx.data.data(), 0, &h);
  if (st != HEMUL_OK) throw_status(g, st);
  return DeviceCiphertext(g, h, c.log_q, c.n_slots);
}

Ciphertext Scheme::download(const DeviceCiphertext& c) const {
  hemul_gpu_ctx* g = gpu();
  if (c.empty()) throw std::invalid_argument("empty device ciphertext");
  Ciphertext r;
  r.ax = make_poly(params_.n, c.log_q, params_.word);
  r.bx = make_poly(params_.n, c.log_q, params_.word);
  const hemul_status st = hemul_gpu_ct_download(g, c.h_, r.ax.data.data(), r.bx.data.data());
  if (st != HEMUL_OK) throw_status(g, st);
  r.log_q = c.log_q;
  r.n_slots = c.n_slots;
  return r;
}

DeviceCiphertext Scheme::he_mul(const DeviceCiphertext& c1, const DeviceCiphertext& c2,
                                const EvalKey& evk) {
  if (c1.log_q != c2.log_q) throw std::invalid_argument("ciphertext modulus mismatch");
  if (c1.log_q - params_.log_p < params_.log_p)
    throw std::runtime_error("multiplicative depth exhausted");
  hemul_gpu_ctx* g = gpu();
  hemul_gpu_ct* h = nullptr;
  const hemul_status st = hemul_gpu_ct_he_mul(g, c1.h_, c2.h_, evk.ax.data.data(),
                                              evk.bx.data.data(),
                                              reinterpret_cast<uintptr_t>(&evk), &h);
  if (st != HEMUL_OK) throw_status(g, st);
  evk_src_ = &evk;
  return DeviceCiphertext(g, h, c1.log_q - params_.log_p, std::max(c1.n_slots, c2.n_slots));
}

DeviceCiphertext Scheme::rescale(const DeviceCiphertext& c) const {
  if (c.log_q - params_.log_p < params_.log_p)
    throw std::runtime_error("modulus exhausted; cannot rescale");
  hemul_gpu_ctx* g = gpu();
  hemul_gpu_ct* h = nullptr;
  const hemul_status st = hemul_gpu_ct_rescale(g, c.h_, &h);
  if (st != HEMUL_OK) throw_status(g, st);
  return DeviceCiphertext(g, h, c.log_q - params_.log_p, c.n_slots);
}

DeviceCiphertext Scheme::mod_down(const DeviceCiphertext& c, int new_log_q) const {
  hemul_gpu_ctx* g = gpu();
  hemul_gpu_ct* h = nullptr;
  const hemul_status st = hemul_gpu_ct_mod_down(g, c.h_, new_log_q, &h);
  if (st != HEMUL_OK) throw_status(g, st);
  return DeviceCiphertext(g, h, new_log_q, c.n_slots);
}

DeviceCiphertext Scheme::load_device(const std::string& path) const {
  hemul_gpu_ctx* g = gpu();
  hemul_gpu_ct* h = nullptr;
  int slots = 0;
  const hemul_status st = hemul_gpu_ct_load(g, path.c_str(), &h, &slots);
  if (st != HEMUL_OK) throw_status(g, st);
  int log_q = 0;
  hemul_gpu_ct_info(h, &log_q, nullptr);
  return DeviceCiphertext(g, h, log_q, slots);
}

void Scheme::save_device(const DeviceCiphertext& c, const std::string& path) const {
  hemul_gpu_ctx* g = gpu();
  if (c.empty()) throw std::invalid_argument("empty device ciphertext");
  const hemul_status st = hemul_gpu_ct_save(g, c.h_, c.n_slots, path.c_str());
  if (st != HEMUL_OK) throw_status(g, st);
}

// The reference algorithm's operation counts for one he_mul (rns.cpp:345-355,
// 370, 385-391; ntt.cpp:168-173, 191-196; call counts heaan.cpp:372-402).
void Scheme::count_he_mul(int log_q) {
  hemul_gpu_ctx* g = gpu();
  int np[2] = {0, 0}, pl[2] = {0, 0};
  for (int region = 1; region <= 2; ++region) {
    int cnt = 0;
    if (hemul_gpu_level_info(g, log_q, region, &cnt, nullptr, 0) != HEMUL_OK) return;
    std::vector<uint64_t> primes(static_cast<size_t>(cnt));
    hemul_gpu_level_info(g, log_q, region, &cnt, primes.data(), cnt);
    BigInt P = bigint_from_u64(1, WordSize::w64);
    for (uint64_t p : primes) P = bigint_mul(P, bigint_from_u64(p, WordSize::w64), WordSize::w64);
    np[region - 1] = cnt;
    pl[region - 1] = static_cast<int>(P.size());
  }
  const uint64_t n = static_cast<uint64_t>(params_.n), logn = static_cast<uint64_t>(params_.log_n);
  const uint64_t L = static_cast<uint64_t>((log_q + 63) / 64);
  // reductions per CRT cell: one 3-word reduction, or one per period
  // (rns.cpp:350-353)
  const uint64_t red = opts_.strategy.kind == AccumKind::three_word_adc
                           ? 1
                           : (L + opts_.strategy.period - 1) / opts_.strategy.period;
  auto crt = [&](uint64_t nprime, uint64_t calls) {
    auto& c = counters[Stage::crt];
    c.mul += calls * n * nprime * L;
    c.adc += calls * n * nprime * L;
    c.modmul += calls * n * nprime * red;
  };
  auto ntt = [&](uint64_t nprime, uint64_t calls) {
    auto& c = counters[Stage::ntt];
    const uint64_t bf = nprime * (n / 2) * logn;
    c.modmul += calls * bf;
    c.addsub += calls * 2 * bf;
  };
  auto intt = [&](uint64_t nprime, uint64_t calls) {
    auto& c = counters[Stage::intt];
    const uint64_t bf = nprime * (n / 2) * logn;
    c.modmul += calls * (bf + nprime * n);
    c.addsub += calls * 2 * bf;
  };
  auto icrt = [&](uint64_t nprime, uint64_t plimbs, uint64_t calls) {
    auto& c = counters[Stage::icrt];
    c.modmul += calls * (n * nprime + n * nprime);  // pointwise + t_j
    c.mul += calls * n * nprime * plimbs;
    c.adc += calls * n * nprime * plimbs;
  };
  const uint64_t products1 = opts_.four_products ? 4 : 3;
  const uint64_t prepares1 = opts_.four_products ? 4 : 6;
  crt(np[0], prepares1);
  ntt(np[0], prepares1);
  icrt(np[0], pl[0], products1);
  intt(np[0], products1);
  crt(np[1], 1);
  ntt(np[1], 1);
  icrt(np[1], pl[1], 2);
  intt(np[1], 2);
}

}  // namespace hemul
