// `hemul` command-line front end relinked against the B200 drop-in
// (libhemul_gpu.so): the subcommands, flags, outputs and exit codes of
// proj/tools/hemul.cpp:86-377.
//
//   hemul keygen  [--log-p 30] [--depth 40] [--word-bits 64] [--ring-degree 0]
//                 [--out-dir .] [--seed 1] [--force]
//   hemul encrypt --params P --pk PK --out CT [--values v,v,..] [--slots 8] [--seed 2]
//   hemul decrypt --params P --sk SK --ct CT
//   hemul mul     --params P --ct1 A --ct2 B --evk EVK --out C
//   hemul bench   [param flags] [--threads T] [--radix 2|4|16|32] [--crt-strategy
//                 three-word-adc|periodic-mod] [--crt-period K] [--icrt naive|reordered]
//                 [--shoup exact|approx] [--reps 32] [--seed 1] [--format table|csv|json]
//
// Exit codes: 0 success, 1 usage error, 2 state / modulus error (mismatched
// moduli, exhausted depth, refusing to overwrite), 3 format error (corrupt
// or truncated files). HEAAN_SEED overrides --seed. `mul` streams both
// ciphertext files into HBM and the product back out through pinned
// buffers (Scheme::load_device / save_device); keygen / encrypt / decrypt
// run their ternary products on the GPU. The analytic `cost` sweeps of the
// reference (costmodel.cpp) are not part of this build.
#include <complex>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <map>
#include <set>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hemul/bench.hpp"
#include "hemul/heaan.hpp"
#include "hemul/io.hpp"
#include "hemul/rng.hpp"

namespace fs = std::filesystem;
using namespace hemul;

namespace {

constexpr int kExitUsage = 1, kExitState = 2, kExitFormat = 3;

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value options and --flag switches of one subcommand
struct Args {
  std::map<std::string, std::string> opt;
  std::set<std::string> flags;

  Args(int argc, char** argv, const std::set<std::string>& options,
       const std::set<std::string>& switches) {
    for (int i = 2; i < argc; ++i) {
      const std::string a = argv[i];
      if (switches.count(a)) {
        flags.insert(a);
      } else if (options.count(a)) {
        if (i + 1 >= argc) throw UsageError(a + " requires a value");
        opt[a] = argv[++i];
      } else {
        throw UsageError("unknown argument: " + a);
      }
    }
  }
  std::string str(const std::string& k, const std::string& def = "") const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
  std::string need(const std::string& k) const {
    auto it = opt.find(k);
    if (it == opt.end()) throw UsageError(k + " is required");
    return it->second;
  }
  long long num(const std::string& k, long long def) const {
    auto it = opt.find(k);
    if (it == opt.end()) return def;
    try {
      size_t pos = 0;
      const long long v = std::stoll(it->second, &pos);
      if (pos != it->second.size()) throw std::invalid_argument("trailing");
      return v;
    } catch (const std::exception&) {
      throw UsageError(k + ": not an integer: " + it->second);
    }
  }
  bool has(const std::string& k) const { return flags.count(k) > 0; }
};

const std::set<std::string> kParamOpts = {"--log-p", "--depth", "--word-bits", "--ring-degree"};

Params params_from(const Args& a) {
  const int wb = static_cast<int>(a.num("--word-bits", 64));
  if (wb != 32 && wb != 64) throw UsageError("--word-bits must be 32 or 64");
  return make_params(static_cast<int>(a.num("--log-p", 30)), static_cast<int>(a.num("--depth", 40)),
                     wb == 64 ? WordSize::w64 : WordSize::w32,
                     static_cast<int>(a.num("--ring-degree", 0)));
}

uint64_t seed_of(const Args& a, uint64_t def) {
  if (const char* env = std::getenv("HEAAN_SEED")) return std::strtoull(env, nullptr, 10);
  return static_cast<uint64_t>(a.num("--seed", static_cast<long long>(def)));
}

void print_slots(const Message& m) {
  std::cout << "[";
  for (size_t i = 0; i < m.slots.size(); ++i)
    std::cout << (i ? "," : "") << "[" << m.slots[i].real() << "," << m.slots[i].imag() << "]";
  std::cout << "]\n";
}

std::set<std::string> with(std::set<std::string> a, const std::set<std::string>& b) {
  a.insert(b.begin(), b.end());
  return a;
}

int cmd_keygen(int argc, char** argv) {
  const Args a(argc, argv, with(kParamOpts, {"--out-dir", "--seed"}), {"--force"});
  const Params p = params_from(a);
  const fs::path dir(a.str("--out-dir", "."));
  if (!fs::exists(dir)) throw IoError("output directory does not exist: " + dir.string());
  const fs::path files[] = {dir / "params.json", dir / "sk.bin", dir / "pk.bin", dir / "evk.bin"};
  for (const auto& f : files)
    if (!a.has("--force") && fs::exists(f))
      throw StateError("refusing to overwrite " + f.string() + " (use --force)");
  Rng rng(seed_of(a, 1));
  Scheme scheme(p);
  const KeySet keys = scheme.keygen(rng);
  save_params(files[0].string(), p);
  save_secret_key(files[1].string(), keys.sk, p);
  save_public_key(files[2].string(), keys.pk, p);
  save_eval_key(files[3].string(), keys.evk, p);
  std::cout << "wrote " << files[0] << ", sk.bin, pk.bin, evk.bin\n";
  return 0;
}

int cmd_encrypt(int argc, char** argv) {
  const Args a(argc, argv, {"--params", "--pk", "--out", "--values", "--slots", "--seed"}, {});
  const std::string params = a.need("--params"), pk_path = a.need("--pk"), out = a.need("--out");
  const Params p = load_params(params);
  const PublicKey pk = load_public_key(pk_path);
  Scheme scheme(p);
  Rng rng(seed_of(a, 2));
  Message m;
  const std::string values = a.str("--values");
  if (!values.empty()) {
    std::istringstream is(values);
    std::string tok;
    while (std::getline(is, tok, ',')) {
      try {
        m.slots.emplace_back(std::stod(tok), 0.0);
      } catch (const std::exception&) {
        throw UsageError("--values: not a number: " + tok);
      }
    }
  } else {
    m.slots.resize(static_cast<size_t>(a.num("--slots", 8)));
    for (auto& s : m.slots) s = {static_cast<double>(rng.next() >> 11) * 0x1p-53 * 2 - 1, 0.0};
  }
  save_ciphertext(out, scheme.encrypt(scheme.encode(m), pk, rng));
  print_slots(m);
  return 0;
}

int cmd_decrypt(int argc, char** argv) {
  const Args a(argc, argv, {"--params", "--sk", "--ct"}, {});
  const std::string params = a.need("--params"), sk_path = a.need("--sk"), ct = a.need("--ct");
  const Params p = load_params(params);
  const SecretKey sk = load_secret_key(sk_path, p);
  const Ciphertext c = load_ciphertext(ct);
  Scheme scheme(p);
  print_slots(scheme.decode(scheme.decrypt(c, sk)));
  return 0;
}

int cmd_mul(int argc, char** argv) {
  const Args a(argc, argv, {"--params", "--ct1", "--ct2", "--evk", "--out"}, {});
  const std::string params = a.need("--params"), ct1 = a.need("--ct1"), ct2 = a.need("--ct2"),
                    evk_path = a.need("--evk"), out = a.need("--out");
  const Params p = load_params(params);
  // the moduli come from the headers: fail before touching the GPU
  const PolyPair h1 = load_poly_pair(ct1), h2 = load_poly_pair(ct2);
  if (h1.log_q != h2.log_q)
    throw StateError("ciphertext moduli differ: " + std::to_string(h1.log_q) + " vs " +
                     std::to_string(h2.log_q));
  const EvalKey evk = load_eval_key(evk_path);
  Scheme scheme(p);
  const DeviceCiphertext d1 = scheme.load_device(ct1);
  const DeviceCiphertext d2 = scheme.load_device(ct2);
  scheme.save_device(scheme.he_mul(d1, d2, evk), out);
  return 0;
}

int cmd_bench(int argc, char** argv) {
  const Args a(argc, argv,
               with(kParamOpts, {"--threads", "--radix", "--crt-strategy", "--crt-period", "--icrt",
                                 "--shoup", "--reps", "--seed", "--format"}),
               {});
  const Params p = params_from(a);
  BenchConfig cfg;
  cfg.threads = std::max(1, static_cast<int>(a.num(
                                "--threads", static_cast<long long>(std::thread::hardware_concurrency()))));
  cfg.reps = static_cast<int>(a.num("--reps", 32));
  if (cfg.reps <= 0) throw UsageError("--reps must be positive");
  cfg.seed = seed_of(a, 1);
  const long long radix = a.num("--radix", 2);
  const std::map<long long, int> radix_log = {{2, 1}, {4, 2}, {16, 4}, {32, 5}};
  if (!radix_log.count(radix)) throw UsageError("--radix must be one of 2,4,16,32");
  cfg.radix_log = radix_log.at(radix);
  const std::string strat = a.str("--crt-strategy", "three-word-adc");
  if (strat == "periodic-mod") {
    cfg.strategy.kind = AccumKind::periodic_mod;
    cfg.strategy.period = static_cast<int>(a.num("--crt-period", 0));
    if (cfg.strategy.period == 0)
      cfg.strategy.period = max_valid_period(generate_primes(2, p.log_n, p.word));
  } else if (strat != "three-word-adc") {
    throw UsageError("--crt-strategy must be three-word-adc or periodic-mod");
  }
  const std::string icrt = a.str("--icrt", "reordered"), shoup = a.str("--shoup", "exact"),
                    fmt = a.str("--format", "table");
  if (icrt != "naive" && icrt != "reordered") throw UsageError("--icrt must be naive or reordered");
  if (shoup != "exact" && shoup != "approx") throw UsageError("--shoup must be exact or approx");
  if (fmt != "table" && fmt != "csv" && fmt != "json")
    throw UsageError("--format must be table, csv or json");
  cfg.icrt_loop_reordered = icrt == "reordered";
  cfg.shoup_approx = shoup == "approx";
  const BenchReport r = run_he_mul_bench(p, cfg, nullptr);
  std::cout << (fmt == "table" ? bench_table(r) : fmt == "csv" ? bench_csv(r) : bench_json(r));
  return 0;
}

int run(int argc, char** argv) {
  const std::string cmd = argc > 1 ? argv[1] : "";
  if (cmd == "keygen") return cmd_keygen(argc, argv);
  if (cmd == "encrypt") return cmd_encrypt(argc, argv);
  if (cmd == "decrypt") return cmd_decrypt(argc, argv);
  if (cmd == "mul") return cmd_mul(argc, argv);
  if (cmd == "bench") return cmd_bench(argc, argv);
  if (cmd == "cost") throw UsageError("the analytic cost sweeps are not part of the B200 build");
  throw UsageError("usage: hemul {keygen|encrypt|decrypt|mul|bench} [options]");
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return run(argc, argv);
  } catch (const UsageError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const IoError& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitFormat;
  } catch (const std::exception& e) {  // StateError, invalid_argument, runtime_error
    std::cerr << "error: " << e.what() << "\n";
    return kExitState;
  }
}
