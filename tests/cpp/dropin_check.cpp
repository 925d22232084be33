// Drop-in check: code written against the reference's C++ API (namespace
// hemul, include/hemul/*.hpp) compiled against libhemul_gpu.so.
//
//   dropin_check keys  <log_p> <depth> <log_n> <seed> <out_prefix>   (GPU)
//       bench-protocol keygen/encode/encrypt (bench.cpp:60-67); writes
//       c1ax c1bx c2ax c2bx evkax evkbx as raw little-endian u64 files;
//       the ternary products run on the GPU; prints the stage times
//   dropin_check bench <log_p> <depth> <log_n> <seed> <reps>          (GPU)
//       run_he_mul_bench; prints "digest <hex>" and the table
//   dropin_check ladder <log_p> <depth> <log_n> <seed>                (GPU)
//       test_heaan.cpp:143-167: he_mul down the modulus chain, decrypting
//       and decoding after each step; prints "max_err <e>"; exit 1 on > 1e-3
//   dropin_check ladder_dev <log_p> <depth> <log_n> <seed>            (GPU)
//       the ladder on DeviceCiphertext (upload / he_mul / mod_down /
//       download); each step bit-identical to the host-API step
//   dropin_check counters <log_p> <depth> <log_n> <seed> <four> <periodic> (GPU)
//       Scheme::counters of one he_mul (compared with the reference's)
//   dropin_check params <log_p> <depth> <log_n> <path>                 (CPU only)
//       save_params (io.hpp)
//   dropin_check tables <np> <log_n> <log_q> <w32>                    (CPU only)
//       digest of generate_primes / make_{crt,ntt,icrt}_tables (params.hpp)
//   dropin_check errors                                                (GPU)
//       test_heaan.cpp:169-182: modulus mismatch / exhausted depth throw
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "hemul/bench.hpp"
#include "hemul/heaan.hpp"
#include "hemul/io.hpp"

using namespace hemul;

namespace {

Message random_message(int slots, Rng& rng) {
  Message m;
  m.slots.resize(slots);
  for (auto& s : m.slots) {
    const double re = static_cast<double>(rng.next() >> 11) * 0x1p-53 * 2 - 1;
    const double im = static_cast<double>(rng.next() >> 11) * 0x1p-53 * 2 - 1;
    s = {re, im};
  }
  return m;
}

double max_err(const Message& a, const Message& b) {
  double e = 0;
  for (size_t i = 0; i < a.slots.size(); ++i) e = std::max(e, std::abs(a.slots[i] - b.slots[i]));
  return e;
}

void write_poly(const std::string& path, const BigPoly& p) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot write " + path);
  std::fwrite(p.data.data(), sizeof(uint64_t), p.data.size(), f);
  std::fclose(f);
}

int cmd_keys(int log_p, int depth, int log_n, uint64_t seed, const std::string& out) {
  const Params p = make_params(log_p, depth, WordSize::w64, log_n);
  Scheme sch(p);
  sch.gpu();  // context creation outside the timings below
  Rng rng(seed);
  const int ns = std::min(64, p.n / 2);
  using clk = std::chrono::steady_clock;
  const auto t0 = clk::now();
  const KeySet keys = sch.keygen(rng);
  const auto t1k = clk::now();
  const Plaintext t1 = sch.encode(random_message(ns, rng));
  const Plaintext t2 = sch.encode(random_message(ns, rng));
  const auto t2e = clk::now();
  const Ciphertext c1 = sch.encrypt(t1, keys.pk, rng);
  const Ciphertext c2 = sch.encrypt(t2, keys.pk, rng);
  const auto t3 = clk::now();
  const Plaintext back = sch.decrypt(c1, keys.sk);
  const auto t4 = clk::now();
  (void)back;
  auto sec = [](clk::duration d) { return std::chrono::duration<double>(d).count(); };
  std::printf("keygen_s %.4f encode_s %.4f encrypt2_s %.4f decrypt_s %.4f\n", sec(t1k - t0),
              sec(t2e - t1k), sec(t3 - t2e), sec(t4 - t3));
  write_poly(out + "c1ax", c1.ax);
  write_poly(out + "c1bx", c1.bx);
  write_poly(out + "c2ax", c2.ax);
  write_poly(out + "c2bx", c2.bx);
  write_poly(out + "evkax", keys.evk.ax);
  write_poly(out + "evkbx", keys.evk.bx);
  return 0;
}

int cmd_bench(int log_p, int depth, int log_n, uint64_t seed, int reps) {
  BenchConfig cfg;
  cfg.seed = seed;
  cfg.reps = reps;
  const BenchReport r = run_he_mul_bench(make_params(log_p, depth, WordSize::w64, log_n), cfg, nullptr);
  std::printf("digest %016llx\n%s", static_cast<unsigned long long>(r.result_digest),
              bench_table(r).c_str());
  return 0;
}

int cmd_ladder(int log_p, int depth, int log_n, uint64_t seed) {
  const Params p = make_params(log_p, depth, WordSize::w64, log_n);
  Scheme sch(p);
  Rng rng(seed);
  const KeySet keys = sch.keygen(rng);
  Message want = random_message(8, rng);
  Ciphertext acc = sch.encrypt(sch.encode(want), keys.pk, rng);
  double worst = 0;
  for (int step = 0; step < depth - 2; ++step) {
    const Message m = random_message(8, rng);
    Ciphertext c = sch.encrypt(sch.encode(m), keys.pk, rng);
    if (c.log_q > acc.log_q) {  // align moduli before multiplying
      c.ax = poly_mod_down(c.ax, acc.log_q);
      c.bx = poly_mod_down(c.bx, acc.log_q);
      c.log_q = acc.log_q;
    }
    acc = sch.he_mul(acc, c, keys.evk);
    for (size_t i = 0; i < want.slots.size(); ++i) want.slots[i] *= m.slots[i];
    worst = std::max(worst, max_err(sch.decode(sch.decrypt(acc, keys.sk)), want));
  }
  std::printf("max_err %.3e final_log_q %d\n", worst, acc.log_q);
  return worst < 1e-3 && acc.log_q == p.log_q_max - (depth - 2) * p.log_p ? 0 : 1;
}

// The same ladder with the accumulator resident on the GPU (Scheme::upload /
// he_mul / mod_down on DeviceCiphertext): every step must equal the host-API
// step bit for bit, and only the fresh operands cross PCIe.
int cmd_ladder_dev(int log_p, int depth, int log_n, uint64_t seed) {
  const Params p = make_params(log_p, depth, WordSize::w64, log_n);
  Scheme sch(p);
  Rng rng(seed);
  const KeySet keys = sch.keygen(rng);
  Message want = random_message(8, rng);
  Ciphertext acc = sch.encrypt(sch.encode(want), keys.pk, rng);
  DeviceCiphertext dacc = sch.upload(acc);
  double worst = 0;
  int mismatches = 0;
  for (int step = 0; step < depth - 2; ++step) {
    const Message m = random_message(8, rng);
    Ciphertext c = sch.encrypt(sch.encode(m), keys.pk, rng);
    DeviceCiphertext dc = sch.upload(c);
    if (dc.log_q > dacc.log_q) dc = sch.mod_down(dc, dacc.log_q);
    if (c.log_q > acc.log_q) {
      c.ax = poly_mod_down(c.ax, acc.log_q);
      c.bx = poly_mod_down(c.bx, acc.log_q);
      c.log_q = acc.log_q;
    }
    acc = sch.he_mul(acc, c, keys.evk);
    dacc = sch.he_mul(dacc, dc, keys.evk);
    const Ciphertext got = sch.download(dacc);
    if (got.log_q != acc.log_q || !poly_equal(got.ax, acc.ax) || !poly_equal(got.bx, acc.bx))
      ++mismatches;
    for (size_t i = 0; i < want.slots.size(); ++i) want.slots[i] *= m.slots[i];
    worst = std::max(worst, max_err(sch.decode(sch.decrypt(got, keys.sk)), want));
  }
  std::printf("max_err %.3e final_log_q %d mismatches %d\n", worst, dacc.log_q, mismatches);
  return worst < 1e-3 && mismatches == 0 ? 0 : 1;
}

// Scheme::counters after one he_mul (same protocol as oracle/ref_shim.cpp
// ref_counters): 20 numbers {mul, adc, modmul, addsub} x 5 stages.
int cmd_counters(int log_p, int depth, int log_n, uint64_t seed, int four, int periodic) {
  const Params p = make_params(log_p, depth, WordSize::w64, log_n);
  Scheme sch(p);
  sch.options().four_products = four != 0;
  if (periodic) {
    sch.options().strategy.kind = AccumKind::periodic_mod;
    sch.options().strategy.period = 4;
  }
  Rng rng(seed);
  const KeySet keys = sch.keygen(rng);
  Message m;
  m.slots.assign(std::min(8, p.n / 2), {0.5, -0.25});
  const Ciphertext c1 = sch.encrypt(sch.encode(m), keys.pk, rng);
  const Ciphertext c2 = sch.encrypt(sch.encode(m), keys.pk, rng);
  sch.warm_level(p.log_q_max, &keys.evk);
  sch.counters.reset();
  sch.he_mul(c1, c2, keys.evk);
  std::printf("counters");
  for (int s = 0; s < 5; ++s) {
    const OpCounts& c = sch.counters.stage[s];
    std::printf(" %llu %llu %llu %llu", (unsigned long long)c.mul, (unsigned long long)c.adc,
                (unsigned long long)c.modmul, (unsigned long long)c.addsub);
  }
  std::printf("\n");
  return 0;
}

int cmd_errors() {
  const Params p = make_params(30, 4, WordSize::w64, 10);
  Scheme sch(p);
  Rng rng(8);
  const KeySet keys = sch.keygen(rng);
  const Message m = random_message(4, rng);
  const Ciphertext c1 = sch.encrypt(sch.encode(m), keys.pk, rng);
  const Ciphertext c2 = sch.encrypt(sch.encode(m), keys.pk, rng);
  const Ciphertext d1 = sch.he_mul(c1, c2, keys.evk);
  int fails = 0;
  try {
    sch.he_mul(d1, c1, keys.evk);
    ++fails;
  } catch (const std::invalid_argument&) {
  }
  const Ciphertext d2 = sch.he_mul(d1, d1, keys.evk);
  const Ciphertext d3 = sch.he_mul(d2, d2, keys.evk);
  try {
    sch.he_mul(d3, d3, keys.evk);
    ++fails;
  } catch (const std::runtime_error&) {
  }
  std::printf("error checks %s\n", fails ? "FAILED" : "ok");
  return fails;
}


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

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    auto arg = [&](int i) { return std::atoi(argv[i]); };
    if (cmd == "keys" && argc == 7)
      return cmd_keys(arg(2), arg(3), arg(4), std::strtoull(argv[5], nullptr, 10), argv[6]);
    if (cmd == "bench" && argc == 7)
      return cmd_bench(arg(2), arg(3), arg(4), std::strtoull(argv[5], nullptr, 10), arg(6));
    if (cmd == "ladder" && argc == 6)
      return cmd_ladder(arg(2), arg(3), arg(4), std::strtoull(argv[5], nullptr, 10));
    if (cmd == "ladder_dev" && argc == 6)
      return cmd_ladder_dev(arg(2), arg(3), arg(4), std::strtoull(argv[5], nullptr, 10));
    if (cmd == "counters" && argc == 8)
      return cmd_counters(arg(2), arg(3), arg(4), std::strtoull(argv[5], nullptr, 10), arg(6),
                          arg(7));
    if (cmd == "params" && argc == 6) {
      save_params(argv[5], make_params(arg(2), arg(3), WordSize::w64, arg(4)));
      return 0;
    }
    if (cmd == "tables" && argc == 6) {
      std::printf("table_digest %016llx\n",
                  static_cast<unsigned long long>(table_digest(arg(2), arg(3), arg(4), arg(5))));
      return 0;
    }
    if (cmd == "errors") return cmd_errors();
    std::fprintf(stderr, "usage: see the header of tests/cpp/dropin_check.cpp\n");
    return 2;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 3;
  }
}
