// C-ABI implementation (include/hemul_gpu.h): context, level cache, evk
// forms, and the HE Mul orchestration on one CUDA stream.
//
// Pipeline of one batched he_mul (reference: heaan.cpp:339-410), every box a
// kernel of this library:
//   region 1 (np1 primes, target 2^log_q)
//     CRT x4 (ax1 bx1 ax2 bx2) -> fwd NTT (4B rows) -> tensor product
//     (d0 = B1B2, d1 = A1B2 + A2B1, d2 = A1A2) -> iNTT (3B rows) -> iCRT (3B)
//   region 2 (np2 primes, target 2^(log_q + log_Q))
//     CRT(d2) -> fwd NTT -> evk product (cached evk forms) -> iNTT (2B rows)
//     -> iCRT (2B)
//   epilogue: out = R_logp(d + R_logQ(ks)) per component.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <list>
#include <memory>
#include <stdexcept>
#include <utility>
#include <string>
#include <thread>
#include <vector>

#include "../../include/hemul_gpu.h"
#include "kernels.hpp"
#include "level_tables.hpp"

using namespace hemul_gpu;

namespace {

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(ptr);
  }
  // grows (never shrinks); returns false on allocation failure
  bool ensure(size_t want) {
    if (want <= bytes) return true;
    if (ptr) cudaFree(ptr);
    ptr = nullptr;
    bytes = 0;
    if (cudaMalloc(&ptr, want) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    bytes = want;
    return true;
  }
};

// One region's device tables in one basis (word 64: the reference's w64
// primes, F64; word 32: the B200 30-bit basis, F32).
struct RegionDev {
  int word = 64;
  int split_h = 0;  // region 1 operands split at bit h (level_tables.hpp)
  int np = 0;
  int target_bits = 0;
  DevBuf primes, tw, itw, btab, hat, big_p, half_p;
  DevBuf primes_t;  // word 32: inverse NTT constants that output t_j (level_tables.hpp)
  DevBuf primes_m, primes_tm;  // the same, compensating Montgomery products (ntt_blk.cu)
  DevBuf twc, itwc;  // tw / itw in the column pass's shared-slot order (column-major pass A)
  struct Crt {
    int in_bits;
    CrtWeights w;
    std::unique_ptr<DevBuf> buf;
  };
  std::vector<Crt> crt;
  struct CrtTc {
    int bit0, bits;
    CrtTcTable tab;
    std::unique_ptr<DevBuf> buf;
  };
  std::vector<CrtTc> crt_tc;  // int8 tensor-core CRT tables (30-bit basis)
  IcrtTable icrt;
  std::vector<uint64_t> host_primes;
  const CrtWeights* weights(int bits) const {
    for (const auto& c : crt)
      if (c.in_bits == bits) return &c.w;
    return nullptr;
  }
  const CrtTcTable* tc_table(int bit0, int bits) const {
    for (const auto& c : crt_tc)
      if (c.bit0 == bit0 && c.bits == bits && crt_tc_supported(c.tab)) return &c.tab;
    return nullptr;
  }
  template <class F>
  const typename F::Prime* P() const {
    return primes.as<const typename F::Prime>();
  }
  template <class F>
  const typename F::Tw* TW() const {
    return tw.as<const typename F::Tw>();
  }
  template <class F>
  const typename F::Tw* ITW() const {
    return itw.as<const typename F::Tw>();
  }
};

// A tensor-core iCRT / finisher table on the device, with its TMA map.
struct BigTcDev {
  DevBuf btab;
  BigTcTable t;
  int out_bit = 0, out_bits = 0;
};

// Both regions of a level in one basis, and the fused finisher's table.
struct Basis {
  std::unique_ptr<RegionDev> r1, r2;
  bool has_fin = false;
  DevBuf fin_btab;
  Finisher fin;  // fused ModDown + add + rescale table (he_mul levels only)
  // int8 tensor-core forms (30-bit split basis): iCRT of d2 and the finisher
  std::unique_ptr<BigTcDev> icrt_tc, fin_tc;
};

struct Level {
  int log_q = 0;
  Basis basis[2];  // [0]: w64 reference primes, [1]: 30-bit basis
  bool has_evk = false;
  int evk_word = 0;  // basis of the cached evk forms
  bool no_basis32 = false;  // the 30-bit basis cannot cover this level
  uint64_t evk_id = 0;
  DevBuf evk_a;  // 2 x np2 x n NTT forms (ax then bx)
};

struct CudaFail : std::runtime_error {
  hemul_status code;
  CudaFail(hemul_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaFail(e == cudaErrorMemoryAllocation ? HEMUL_E_OOM : HEMUL_E_CUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
  }
}

template <typename T>
void upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
  if (!b.ensure(v.size() * sizeof(T) + 16)) throw CudaFail(HEMUL_E_OOM, "device allocation failed");
  check(cudaMemcpyAsync(b.ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st),
        "table upload");
}

}  // namespace

struct hemul_gpu_ctx {
  int device = 0;
  int log_n = 0, n = 0, log_p = 0, depth = 0, log_q_max = 0;
  cudaStream_t stream = nullptr;      // where every launch goes
  cudaStream_t own_stream = nullptr;  // created by the context
  cudaStream_t h2d = nullptr, d2h = nullptr;  // copy streams of the host-buffer pipeline
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  std::list<std::unique_ptr<Level>> cache;  // most recent first, capacity 2
  std::string err;
  uint64_t launches = 0;
  bool timing = false;
  uint64_t call_id = 0;  // he_mul calls, to attribute stage times
  double stage_ms[HEMUL_STAGE_COUNT] = {};
  double kclass_ms[HEMUL_KCLASS_COUNT] = {};
  uint64_t kclass_launches[HEMUL_KCLASS_COUNT] = {};
  struct Mark {
    int stage, klass;
    uint64_t call;
    cudaEvent_t a, b;
  };
  std::vector<Mark> marks;
  std::vector<cudaEvent_t> event_pool;
  // scratch
  DevBuf in, r1, dpoly, r2, ks, outb, rescale_buf, flagbuf;
  DevBuf r1b, r2b;  // out-of-place NTT pass-A buffers of the transposed layout
  DevBuf tern_a, tern_b, tern_nz;  // mul_by_ternary scratch
  DevBuf evk_tmp;  // the key reduced mod 2^(log_q + log_Q) (30-bit basis, evk_forms)
  void* pinned[2] = {nullptr, nullptr};  // file streaming (hemul_gpu_ct_load / _save)
  cudaEvent_t ev_pin[2] = {nullptr, nullptr};
  int force_exact = 0;  // HEMUL_OPT_FORCE_EXACT (tests the exact fix-up path)
  int basis = 32;       // HEMUL_OPT_BASIS: he_mul prime basis (32 or 64)
  int tensor_cores = 1;  // HEMUL_OPT_TENSOR_CORES: int8 tcgen05 base conversions
  int transposed = 1;    // HEMUL_OPT_TRANSPOSED: column-major RNS rows around pass A
  int level_cache = 2;   // HEMUL_OPT_LEVEL_CACHE: LRU capacity (heaan.cpp:119-150: 2)

  cudaEvent_t take_event() {
    if (!event_pool.empty()) {
      cudaEvent_t e = event_pool.back();
      event_pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    check(cudaEventCreate(&e), "cudaEventCreate");
    return e;
  }
};

namespace {

hemul_status fail(hemul_gpu_ctx* c, hemul_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

template <typename F>
hemul_status guarded(hemul_gpu_ctx* c, F&& f) {
  try {
    if (cudaSetDevice(c->device) != cudaSuccess) {
      cudaGetLastError();
      return fail(c, HEMUL_E_CUDA, "cudaSetDevice failed");
    }
    return f();
  } catch (const CudaFail& e) {
    return fail(c, e.code, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(c, HEMUL_E_ARG, e.what());
  } catch (const std::bad_alloc&) {
    return fail(c, HEMUL_E_OOM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(c, HEMUL_E_ARG, e.what());
  }
}

// Runs one launch (or copy) f() on the context stream; with timing on, the
// launch is bracketed by CUDA events and attributed to a reference stage
// bucket (counters.hpp:13, ScopedStageTimer counters.hpp:58-76) and to a
// kernel class. Events are read back lazily (flush_marks).
template <typename F>
void run_on(hemul_gpu_ctx* c, cudaStream_t st, int stage, int klass, const char* what, F&& f) {
  cudaEvent_t a = nullptr;
  if (c->timing) {
    a = c->take_event();
    check(cudaEventRecord(a, st), "event");
  }
  check(f(), what);
  if (klass < HEMUL_KCLASS_H2D) ++c->launches;
  if (c->timing) {
    cudaEvent_t b = c->take_event();
    check(cudaEventRecord(b, st), "event");
    c->marks.push_back({stage, klass, c->call_id, a, b});
  }
}

template <typename F>
void run(hemul_gpu_ctx* c, int stage, int klass, const char* what, F&& f) {
  run_on(c, c->stream, stage, klass, what, f);
}

// Reads back every pending event pair: stage times of the latest he_mul and
// cumulative per-kernel-class times.
void flush_marks(hemul_gpu_ctx* c) {
  if (c->marks.empty()) return;
  check(cudaStreamSynchronize(c->stream), "timing sync");
  bool fresh = false;
  for (auto& m : c->marks) {
    float ms = 0;
    cudaEventSynchronize(m.b);  // copies run on their own streams
    cudaEventElapsedTime(&ms, m.a, m.b);
    if (m.call == c->call_id) {
      if (!fresh) {
        for (double& v : c->stage_ms) v = 0;
        fresh = true;
      }
      c->stage_ms[m.stage] += ms;
    }
    c->kclass_ms[m.klass] += ms;
    ++c->kclass_launches[m.klass];
    c->event_pool.push_back(m.a);
    c->event_pool.push_back(m.b);
  }
  c->marks.clear();
}

void fill_region(RegionDev& d, const RegionHost& h, cudaStream_t st) {
  d.word = h.word;
  d.split_h = h.split_h;
  d.np = h.np;
  d.target_bits = h.target_bits;
  d.host_primes = h.primes;
  if (h.word == 64) {
    upload(d.primes, h.dev, st);
    upload(d.tw, h.tw, st);
    upload(d.itw, h.itw, st);
  } else {
    upload(d.primes, h.dev32, st);
    upload(d.primes_t, h.dev32_t, st);
    upload(d.primes_m, h.dev32_m, st);
    upload(d.primes_tm, h.dev32_tm, st);
    // twiddles on the device (tables.cu): primes, psi_j, psi_j^-1 in, np x n
    // Shoup pairs per direction out
    const size_t n = size_t(1) << h.log_n, bytes = size_t(h.np) * n * sizeof(Twiddle32);
    if (!d.tw.ensure(bytes + 16) || !d.itw.ensure(bytes + 16))
      throw CudaFail(HEMUL_E_OOM, "device allocation failed");
    std::vector<uint32_t> pr(3 * size_t(h.np));
    for (int j = 0; j < h.np; ++j) {
      const uint64_t p = h.primes[j];
      pr[j] = uint32_t(p);
      pr[h.np + j] = uint32_t(h.roots[j]);
      pr[2 * h.np + j] = uint32_t(h.roots_inv[j]);
    }
    DevBuf tmp;
    upload(tmp, pr, st);
    const uint32_t* t = tmp.as<uint32_t>();
    check(build_twiddles32(t, t + h.np, t + 2 * h.np, h.np, h.log_n, d.tw.as<Twiddle32>(),
                           d.itw.as<Twiddle32>(), st),
          "twiddle tables");
    const int S = ntt_pass_a_levels(h.log_n);
    if (ntt_col_transposed_supported(h.log_n, S)) {
      for (auto [src, dst] : {std::pair{&d.tw, &d.twc}, std::pair{&d.itw, &d.itwc}}) {
        if (!dst->ensure((size_t(h.np) << S) * sizeof(Twiddle32) + 16))
          throw CudaFail(HEMUL_E_OOM, "device allocation failed");
        check(ntt_col_slot_twiddles(src->as<Twiddle32>(), h.np, h.log_n, S, dst->as<Twiddle32>(),
                                    st),
              "slot twiddles");
      }
    }
    check(cudaStreamSynchronize(st), "twiddle tables");  // tmp is freed on return
  }
  upload(d.btab, h.btab, st);
  d.icrt.btab = d.btab.as<uint32_t>();
  d.icrt.m_out = h.m_out;
  d.icrt.m_pad = h.m_pad;
  d.icrt.target_bits = h.target_bits;
  upload(d.hat, h.hat_full, st);
  upload(d.big_p, h.big_p, st);
  upload(d.half_p, h.half_p, st);
  d.icrt.hat = d.hat.as<uint64_t>();
  d.icrt.big_p = d.big_p.as<uint64_t>();
  d.icrt.half_p = d.half_p.as<uint64_t>();
  d.icrt.p_limbs = h.p_limbs;
  d.crt.clear();
  for (const auto& c : h.crt) {
    RegionDev::Crt dc;
    dc.in_bits = c.in_bits;
    dc.buf = std::make_unique<DevBuf>();
    upload(*dc.buf, c.wtab, st);
    dc.w.wtab = dc.buf->as<uint32_t>();
    dc.w.chunks = c.chunks;
    dc.w.ld = c.ld;
    d.crt.push_back(std::move(dc));
  }
  d.crt_tc.clear();
  for (const auto& t : h.crt_tc) {
    RegionDev::CrtTc dt;
    dt.bit0 = t.bit0;
    dt.bits = t.bits;
    dt.buf = std::make_unique<DevBuf>();
    upload(*dt.buf, t.btab, st);
    dt.tab.btab = dt.buf->as<uint8_t>();
    dt.tab.kpad = t.kpad;
    dt.tab.col_tile = t.col_tile;
    dt.tab.ncol_tiles = t.ncol_tiles;
    dt.tab.primes_per_tile = t.primes_per_tile;
    dt.tab.limb0 = t.limb0;
    dt.tab.end_bit = t.end_bit;
    d.crt_tc.push_back(std::move(dt));
  }
}

// cuTensorMapEncodeTiled, resolved through the runtime (no libcuda link).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn)
      throw CudaFail(HEMUL_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  return encode;
}

// 2-D TMA map of a u32 residue array [rows][n], boxes of 128 residues x 16
// rows, no swizzle (bigint_tc.cu's t rows).
void make_raw_tmap(CUtensorMap* m, const uint32_t* g, uint64_t n, uint64_t rows) {
  const cuuint64_t dims[2] = {n, rows};
  const cuuint64_t strides[1] = {n * 4};
  const cuuint32_t box[2] = {128, 16};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = tmap_encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, const_cast<uint32_t*>(g),
                                    dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaFail(HEMUL_E_CUDA, "cuTensorMapEncodeTiled (t rows) failed");
}

std::unique_ptr<BigTcDev> upload_bigint(const BigTcHost& h, cudaStream_t st) {
  if (!bigint_tc_supported(h.n_cols)) return nullptr;
  auto d = std::make_unique<BigTcDev>();
  upload(d->btab, h.btab, st);
  BigTcTable& t = d->t;
  t.btab = d->btab.as<uint8_t>();
  t.n_cols = h.n_cols;
  t.k_bytes = h.k_bytes;
  t.k_slot = h.k_slot;
  t.nseg = h.nseg;
  for (int s = 0; s < 3; ++s) {
    t.slot0[s] = h.slot0[s];
    t.np[s] = h.np[s];
  }
  d->out_bit = h.out_bit;
  d->out_bits = h.out_bits;
  return d;
}

int host_threads() {
  const unsigned t = std::thread::hardware_concurrency();
  return t ? int(t < 32 ? t : 32) : 1;
}

// Scheme::level (heaan.cpp:119-150): LRU of capacity 2 keyed by log_q. The
// tables of each basis are built on first use (get_basis).
Level& get_level(hemul_gpu_ctx* c, int log_q) {
  for (auto it = c->cache.begin(); it != c->cache.end(); ++it)
    if ((*it)->log_q == log_q) {
      c->cache.splice(c->cache.begin(), c->cache, it);
      return *c->cache.front();
    }
  if (log_q <= 0 || log_q > c->log_q_max) throw std::invalid_argument("log_q out of range");
  auto lv = std::make_unique<Level>();
  lv->log_q = log_q;
  c->cache.push_front(std::move(lv));
  while (c->cache.size() > size_t(c->level_cache)) c->cache.pop_back();
  return *c->cache.front();
}

// Regions 1 and 2 of a level in basis `word` (64 or 32), plus the finisher
// table when he_mul can run at this level. Throws std::runtime_error when
// the 30-bit basis has too few primes for the ring degree.
int evk_bits(const hemul_gpu_ctx* c, int log_q, int word);

Basis& get_basis(hemul_gpu_ctx* c, Level& lv, int word) {
  Basis& b = lv.basis[word == 64 ? 0 : 1];
  if (b.r1) return b;
  const int log_q = lv.log_q;
  const int th = host_threads();
  // the 30-bit basis splits region-1 operands in halves (h = ceil(log_q / 2))
  const int split_h = word == 32 ? split_point(log_q) : 0;
  RegionHost h1 = build_region(1, log_q, c->log_q_max, c->log_n, {log_q}, th, word, split_h);
  RegionHost h2 = build_region(2, log_q, c->log_q_max, c->log_n,
                               {log_q, evk_bits(c, log_q, word)}, th, word);
  auto r1 = std::make_unique<RegionDev>();
  auto r2 = std::make_unique<RegionDev>();
  fill_region(*r1, h1, c->stream);
  fill_region(*r2, h2, c->stream);
  if (log_q - c->log_p >= c->log_p) {  // a level he_mul can run at
    const FinisherHost fh = build_finisher(h1, h2, log_q, c->log_q_max, c->log_p);
    upload(b.fin_btab, fh.btab, c->stream);
    Finisher& f = b.fin;
    f.btab = b.fin_btab.as<uint32_t>();
    f.cols = fh.cols;
    f.cols_pad = fh.cols_pad;
    f.k2 = fh.k2;
    f.k1 = fh.k1;
    f.base = fh.base;
    f.half_q_bit = fh.half_q_bit;
    f.half_p_bit = fh.half_p_bit;
    f.out_bit = fh.out_bit;
    f.out_bits = fh.out_bits;
    f.log_q = log_q;
    f.log_Q = c->log_q_max;
    f.log_p = c->log_p;
    f.split_h = split_h;
    b.has_fin = true;
    if (word == 32 && split_h % 8 == 0)
      b.fin_tc = upload_bigint(build_finisher_tc(h1, h2, log_q, c->log_q_max, c->log_p), c->stream);
  }
  if (word == 32 && split_h % 8 == 0) b.icrt_tc = upload_bigint(build_icrt_tc(h1), c->stream);
  check(cudaStreamSynchronize(c->stream), "level upload");
  b.r1 = std::move(r1);
  b.r2 = std::move(r2);
  return b;
}

// The basis he_mul runs in: the context's choice, or the reference's w64
// primes when the 30-bit basis cannot cover the level (fields.cuh).
int mul_word(hemul_gpu_ctx* c, Level& lv) {
  if (c->basis == 64) return 64;
  if (lv.no_basis32) return 64;
  try {
    get_basis(c, lv, 32);
    return 32;
  } catch (const BasisUnavailable&) {  // too few 30-bit primes; CUDA errors propagate
    Basis& b = lv.basis[1];
    b.r1.reset();
    b.r2.reset();
    b.icrt_tc.reset();
    b.fin_tc.reset();
    b.fin_btab.reset();
    b.has_fin = false;
    lv.no_basis32 = true;
    return 64;
  }
}

bool is_device(const hemul_gpu_ctx* c, const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice) {
    if (a.device != c->device) throw std::invalid_argument("device pointer on another GPU");
    return true;
  }
  cudaGetLastError();
  return false;
}

void ensure(DevBuf& b, size_t bytes) {
  if (!b.ensure(bytes)) throw CudaFail(HEMUL_E_OOM, "device allocation failed");
}

int limbs_of(int bits) { return (bits + 63) / 64; }

// Bits of the evk coefficients the region-2 CRT takes: the reference's full
// 2 log_Q (w64 basis) or the key reduced mod 2^(log_q + log_Q) (30-bit basis,
// see evk_forms and build_region).
int evk_bits(const hemul_gpu_ctx* c, int log_q, int word) {
  return word == 64 ? 2 * c->log_q_max : log_q + c->log_q_max;
}

// Forward NTT of `rows` rows, one launch per memory pass (only the first
// `passes` of them when a fused middle pass follows).
template <class F>
void ntt_fwd(hemul_gpu_ctx* c, const RegionDev& r, typename F::W* data, size_t rows, int stage,
             int passes = 2) {
  const int total = ntt_num_passes(c->log_n);
  for (int pass = 0; pass < total && pass < passes; ++pass)
    run(c, stage, pass == 0 ? HEMUL_KCLASS_NTT_A : HEMUL_KCLASS_NTT_B, "NTT", [&] {
      return ntt_forward_pass<F>(pass, data, rows, r.np, c->log_n, r.TW<F>(), r.P<F>(),
                                 c->stream);
    });
}

// Inverse NTT; passes = 1 runs only the final pass (after a fused middle pass).
// to_t (30-bit basis): the last level scales by n^-1 (P/p_j)^-1, giving the
// tensor-core iCRT / finisher operand t_j instead of x_j. mont: the data are
// Montgomery products x y 2^-32 (ntt_blk.cu middle pass); the last level
// multiplies the 2^32 back in.
template <class F>
void ntt_inv(hemul_gpu_ctx* c, const RegionDev& r, typename F::W* data, size_t rows, int stage,
             int passes = 2, bool to_t = false, bool mont = false) {
  const int total = ntt_num_passes(c->log_n);
  const typename F::Prime* pr =
      mont ? (to_t ? r.primes_tm : r.primes_m).as<const typename F::Prime>()
           : to_t ? r.primes_t.as<const typename F::Prime>() : r.P<F>();
  for (int pass = total > passes ? total - passes : 0; pass < total; ++pass)
    run(c, stage, pass + 1 == total ? HEMUL_KCLASS_INTT_A : HEMUL_KCLASS_INTT_B, "iNTT", [&] {
      return ntt_inverse_pass<F>(pass, data, rows, r.np, c->log_n, r.ITW<F>(), pr, c->stream);
    });
}

// Stages a caller buffer on the device when it is host memory.
const uint64_t* stage_in(hemul_gpu_ctx* c, const uint64_t* p, size_t words, uint64_t* scratch) {
  if (is_device(c, p)) return p;
  run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_H2D, "H2D",
      [&] { return cudaMemcpyAsync(scratch, p, words * 8, cudaMemcpyDefault, c->stream); });
  return scratch;
}

// Scheme::level's evk transforms (heaan.cpp:152-167): CRT of the key polys
// into the region-2 primes of the he_mul basis + forward NTT, kept on the
// device. The 30-bit basis first reduces the 2 log_Q-bit key mod
// 2^(log_q + log_Q) (poly_mod_down on the device): the key-switch product is
// only used mod qQ, so the result is unchanged and region 2 needs
// 2 log_q + log_Q + log_n bits instead of log_q + 2 log_Q + log_n.
template <class F>
void evk_forms(hemul_gpu_ctx* c, Level& lv, const RegionDev& r2, const uint64_t* a,
               const uint64_t* b) {
  using W = typename F::W;
  const size_t n = size_t(c->n);
  ensure(lv.evk_a, 2 * size_t(r2.np) * n * sizeof(W));  // [evk_ax form | evk_bx form]
  const int bits = evk_bits(c, lv.log_q, sizeof(W) == 8 ? 64 : 32);
  const CrtWeights* w = r2.weights(bits);
  W* fa = lv.evk_a.as<W>();
  W* fb = fa + size_t(r2.np) * n;
  const int Le = limbs_of(bits);
  if (bits < 2 * c->log_q_max) {
    ensure(c->evk_tmp, 2 * n * Le * 8);
    uint64_t* ra = c->evk_tmp.as<uint64_t>();
    uint64_t* rb = ra + n * Le;
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "evk mod_down", [&] {
      const cudaError_t e = mod_down(a, ra, 1, c->log_n, 2 * c->log_q_max, bits, c->stream);
      return e != cudaSuccess ? e : mod_down(b, rb, 1, c->log_n, 2 * c->log_q_max, bits, c->stream);
    });
    a = ra;
    b = rb;
  }
  run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_CRT, "evk CRT", [&] {
    return crt_forward<F>(a, Le, 1, c->log_n, *w, r2.P<F>(), r2.np, fa, c->stream);
  });
  run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_CRT, "evk CRT", [&] {
    return crt_forward<F>(b, Le, 1, c->log_n, *w, r2.P<F>(), r2.np, fb, c->stream);
  });
  ntt_fwd<F>(c, r2, fa, 2 * size_t(r2.np), HEMUL_STAGE_EXTRA);
}

void set_evk_forms(hemul_gpu_ctx* c, Level& lv, const uint64_t* evk_ax, const uint64_t* evk_bx,
                   uint64_t id) {
  const size_t n = size_t(c->n);
  const int Le = limbs_of(2 * c->log_q_max);
  const int word = mul_word(c, lv);
  const RegionDev& r2 = *get_basis(c, lv, word).r2;
  ensure(c->in, 2 * n * Le * 8);
  const uint64_t* a = stage_in(c, evk_ax, n * Le, c->in.as<uint64_t>());
  const uint64_t* b = stage_in(c, evk_bx, n * Le, c->in.as<uint64_t>() + n * Le);
  if (word == 64)
    evk_forms<F64>(c, lv, r2, a, b);
  else
    evk_forms<F32>(c, lv, r2, a, b);
  check(cudaStreamSynchronize(c->stream), "evk forms");
  lv.has_evk = true;
  lv.evk_word = word;
  lv.evk_id = id;
}

// Output buffers: the caller's device buffers, or scratch + D2H.
struct OutPair {
  uint64_t* a;
  uint64_t* b;
  bool device;
};

OutPair out_pair(hemul_gpu_ctx* c, uint64_t* oa, uint64_t* ob, size_t words, DevBuf& scratch) {
  if (is_device(c, oa) && is_device(c, ob)) return {oa, ob, true};
  ensure(scratch, 2 * words * 8);
  return {scratch.as<uint64_t>(), scratch.as<uint64_t>() + words, false};
}

void copy_out(hemul_gpu_ctx* c, const OutPair& o, uint64_t* oa, uint64_t* ob, size_t words) {
  if (o.device) return;
  run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H",
      [&] { return cudaMemcpyAsync(oa, o.a, words * 8, cudaMemcpyDefault, c->stream); });
  run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H",
      [&] { return cudaMemcpyAsync(ob, o.b, words * 8, cudaMemcpyDefault, c->stream); });
  check(cudaStreamSynchronize(c->stream), "D2H");
}

// Stage checkpoint of he_mul_device (hemul_gpu_he_mul_trace): the run stops
// after checkpoint `stop` and copies that stage's device buffer to dst.
struct Trace {
  int stop = 0;
  void* dst = nullptr;
  size_t cap = 0;
  size_t written = 0;
};

template <class F>
void he_mul_device(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                   const uint64_t* const in[4], uint64_t* out_ax, uint64_t* out_bx,
                   Trace* tr = nullptr);
void he_mul_any(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                const uint64_t* const in[4], uint64_t* out_ax, uint64_t* out_bx);
void he_mul_pipelined(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                      const uint64_t* const src[4], bool dev_in, uint64_t* out_ax,
                      uint64_t* out_bx, bool dev_out);

}  // namespace

extern "C" {

hemul_status hemul_gpu_create(int device, int log_p, int depth, int log_n_override,
                              hemul_gpu_ctx** out) {
  if (!out) return HEMUL_E_ARG;
  *out = nullptr;
  if (log_p <= 0 || depth <= 0) return HEMUL_E_ARG;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return HEMUL_E_CUDA;
  }
  if (device < 0 || device >= count) return HEMUL_E_ARG;
  auto c = std::make_unique<hemul_gpu_ctx>();
  c->device = device;
  c->log_p = log_p;
  c->depth = depth;
  c->log_q_max = log_p * depth;  // params.cpp:70
  if (log_n_override) {
    c->log_n = log_n_override;
  } else {  // params.cpp:56-62
    const int q = c->log_q_max;
    if (q <= 300) c->log_n = 14;
    else if (q <= 600) c->log_n = 15;
    else if (q <= 1200) c->log_n = 16;
    else if (q <= 2400) c->log_n = 17;
    else return HEMUL_E_ARG;  // "modulus too large for security table"
  }
  if (c->log_n < 7 || c->log_n > 17) return HEMUL_E_ARG;
  c->n = 1 << c->log_n;
  if (cudaSetDevice(device) != cudaSuccess) return HEMUL_E_CUDA;
  if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess)
    return HEMUL_E_CUDA;
  c->stream = c->own_stream;
  if (cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking) != cudaSuccess)
    return HEMUL_E_CUDA;
  for (int s = 0; s < 2; ++s)
    if (cudaEventCreateWithFlags(&c->ev_h2d[s], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_comp[s], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c->ev_d2h[s], cudaEventDisableTiming) != cudaSuccess)
      return HEMUL_E_CUDA;
  // keep freed stream-ordered memory (device ciphertext handles) in the pool
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  cudaGetLastError();
  if (ntt_setup_attributes() != cudaSuccess || crt_setup_attributes() != cudaSuccess ||
      crt_tc_setup_attributes() != cudaSuccess || bigint_tc_setup_attributes() != cudaSuccess ||
      icrt_setup_attributes() != cudaSuccess)
    return HEMUL_E_CUDA;
  *out = c.release();
  return HEMUL_OK;
}

void hemul_gpu_destroy(hemul_gpu_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (auto& m : c->marks) {
    cudaEventDestroy(m.a);
    cudaEventDestroy(m.b);
  }
  for (auto e : c->event_pool) cudaEventDestroy(e);
  c->cache.clear();
  cudaStreamSynchronize(c->h2d);
  cudaStreamSynchronize(c->d2h);
  for (int s = 0; s < 2; ++s) {
    cudaEventDestroy(c->ev_h2d[s]);
    cudaEventDestroy(c->ev_comp[s]);
    cudaEventDestroy(c->ev_d2h[s]);
  }
  for (int s = 0; s < 2; ++s) {
    if (c->pinned[s]) cudaFreeHost(c->pinned[s]);
    if (c->ev_pin[s]) cudaEventDestroy(c->ev_pin[s]);
  }
  cudaStreamDestroy(c->h2d);
  cudaStreamDestroy(c->d2h);
  cudaStreamDestroy(c->own_stream);
  delete c;
}

const char* hemul_gpu_last_error(const hemul_gpu_ctx* c) { return c ? c->err.c_str() : ""; }

hemul_status hemul_gpu_params(const hemul_gpu_ctx* c, int out[5]) {
  if (!c || !out) return HEMUL_E_ARG;
  out[0] = c->log_n;
  out[1] = c->n;
  out[2] = c->log_p;
  out[3] = c->depth;
  out[4] = c->log_q_max;
  return HEMUL_OK;
}

hemul_status hemul_gpu_set_stream(hemul_gpu_ctx* c, void* stream) {
  if (!c) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check(cudaStreamSynchronize(c->stream), "stream switch");
    c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_set_level(hemul_gpu_ctx* c, int log_q) {
  if (!c) return HEMUL_E_ARG;
  return guarded(c, [&] {
    Level& lv = get_level(c, log_q);
    get_basis(c, lv, mul_word(c, lv));
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_set_evk(hemul_gpu_ctx* c, int log_q, const uint64_t* evk_ax,
                               const uint64_t* evk_bx, uint64_t evk_id) {
  if (!c || !evk_ax || !evk_bx) return HEMUL_E_ARG;
  return guarded(c, [&] {
    Level& lv = get_level(c, log_q);
    set_evk_forms(c, lv, evk_ax, evk_bx, evk_id);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_level_info(hemul_gpu_ctx* c, int log_q, int region, int* np,
                                  uint64_t* primes, int cap) {
  if (!c || (region != 1 && region != 2 && region != -1 && region != -2)) return HEMUL_E_ARG;
  return guarded(c, [&] {
    if (log_q <= 0 || log_q > c->log_q_max) throw std::invalid_argument("log_q out of range");
    if (region > 0) {  // the reference's rule, host arithmetic only (no tables)
      const std::vector<uint64_t> ps =
          reference_primes(region, log_q, c->log_q_max, c->log_n, nullptr);
      if (np) *np = static_cast<int>(ps.size());
      for (int j = 0; j < int(ps.size()) && j < cap && primes; ++j) primes[j] = ps[j];
      return HEMUL_OK;
    }
    Level& lv = get_level(c, log_q);
    const Basis& b = get_basis(c, lv, mul_word(c, lv));
    const RegionDev& r = region == -1 ? *b.r1 : *b.r2;
    if (np) *np = r.np;
    for (int j = 0; j < r.np && j < cap && primes; ++j) primes[j] = r.host_primes[j];
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_set_option(hemul_gpu_ctx* c, int option, int value) {
  if (!c) return HEMUL_E_ARG;
  switch (option) {
    case HEMUL_OPT_FORCE_EXACT:
      c->force_exact = value != 0;
      return HEMUL_OK;
    case HEMUL_OPT_TENSOR_CORES:
      c->tensor_cores = value != 0;
      return HEMUL_OK;
    case HEMUL_OPT_TRANSPOSED:
      c->transposed = value != 0;
      return HEMUL_OK;
    case HEMUL_OPT_LEVEL_CACHE:
      if (value < 1 || value > 1024) return fail(c, HEMUL_E_ARG, "level cache capacity out of range");
      c->level_cache = value;
      while (c->cache.size() > size_t(c->level_cache)) c->cache.pop_back();
      return HEMUL_OK;
    case HEMUL_OPT_BASIS:
      if (value != 32 && value != 64) return fail(c, HEMUL_E_ARG, "basis must be 32 or 64");
      c->basis = value;
      return HEMUL_OK;
    default:
      return fail(c, HEMUL_E_ARG, "unknown option");
  }
}

hemul_status hemul_gpu_enable_stage_timing(hemul_gpu_ctx* c, int on) {
  if (!c) return HEMUL_E_ARG;
  c->timing = on != 0;
  return HEMUL_OK;
}

hemul_status hemul_gpu_stage_ms(hemul_gpu_ctx* c, double ms[HEMUL_STAGE_COUNT]) {
  if (!c || !ms) return HEMUL_E_ARG;
  return guarded(c, [&] {
    flush_marks(c);
    for (int i = 0; i < HEMUL_STAGE_COUNT; ++i) ms[i] = c->stage_ms[i];
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_kernel_stats(hemul_gpu_ctx* c, double ms[HEMUL_KCLASS_COUNT],
                                    uint64_t launches[HEMUL_KCLASS_COUNT]) {
  if (!c) return HEMUL_E_ARG;
  return guarded(c, [&] {
    flush_marks(c);
    for (int i = 0; i < HEMUL_KCLASS_COUNT; ++i) {
      if (ms) ms[i] = c->kclass_ms[i];
      if (launches) launches[i] = c->kclass_launches[i];
    }
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_reset_stats(hemul_gpu_ctx* c) {
  if (!c) return HEMUL_E_ARG;
  return guarded(c, [&] {
    flush_marks(c);
    for (int i = 0; i < HEMUL_KCLASS_COUNT; ++i) {
      c->kclass_ms[i] = 0;
      c->kclass_launches[i] = 0;
    }
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_imad_peak(hemul_gpu_ctx* c, double* ops_per_s) {
  if (!c || !ops_per_s) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check(imad_peak(ops_per_s, c->stream), "IMAD probe");
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_tc_peak(hemul_gpu_ctx* c, double* ops_per_s) {
  if (!c || !ops_per_s) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check(tc_peak(ops_per_s, c->stream), "tensor-core probe");
    return HEMUL_OK;
  });
}

uint64_t hemul_gpu_launch_count(const hemul_gpu_ctx* c) { return c ? c->launches : 0; }

hemul_status hemul_gpu_synchronize(hemul_gpu_ctx* c) {
  if (!c) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check(cudaStreamSynchronize(c->stream), "synchronize");
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_he_mul(hemul_gpu_ctx* c, int c1_log_q, int c2_log_q, size_t batch,
                              const uint64_t* c1_ax, const uint64_t* c1_bx,
                              const uint64_t* c2_ax, const uint64_t* c2_bx,
                              const uint64_t* evk_ax, const uint64_t* evk_bx, uint64_t evk_id,
                              uint64_t* out_ax, uint64_t* out_bx) {
  if (!c) return HEMUL_E_ARG;
  // heaan.cpp:341-345, same order and messages
  if (c1_log_q != c2_log_q)
    return fail(c, HEMUL_E_MODULUS_MISMATCH, "ciphertext modulus mismatch");
  const int log_q = c1_log_q;
  if (log_q - c->log_p < c->log_p)
    return fail(c, HEMUL_E_DEPTH, "multiplicative depth exhausted");
  if (batch == 0) return HEMUL_OK;
  if (!c1_ax || !c1_bx || !c2_ax || !c2_bx || !out_ax || !out_bx)
    return fail(c, HEMUL_E_ARG, "null buffer");
  return guarded(c, [&]() -> hemul_status {
    Level& lv = get_level(c, log_q);
    const int word = mul_word(c, lv);
    if (evk_ax && evk_bx &&
        (!lv.has_evk || evk_id == 0 || lv.evk_id != evk_id || lv.evk_word != word))
      set_evk_forms(c, lv, evk_ax, evk_bx, evk_id);
    if (!lv.has_evk || lv.evk_word != word)
      return fail(c, HEMUL_E_NO_EVK, "evaluation key not set for this level");
    ++c->call_id;
    const uint64_t* src[4] = {c1_ax, c1_bx, c2_ax, c2_bx};
    bool dev_in = true;
    for (const uint64_t* s : src) dev_in = dev_in && is_device(c, s);
    const bool dev_out = is_device(c, out_ax) && is_device(c, out_bx);
    if (dev_in && dev_out) {
      he_mul_any(c, lv, log_q, batch, src, out_ax, out_bx);
      return HEMUL_OK;
    }
    he_mul_pipelined(c, lv, log_q, batch, src, dev_in, out_ax, out_bx, dev_out);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_engine_info(hemul_gpu_ctx* c, int log_q, int info[HEMUL_INFO_COUNT]) {
  if (!c || !info) return HEMUL_E_ARG;
  return guarded(c, [&] {
    Level& lv = get_level(c, log_q);
    const int word = mul_word(c, lv);
    const Basis& bs = get_basis(c, lv, word);
    const RegionDev& r1 = *bs.r1;
    const RegionDev& r2 = *bs.r2;
    const bool tc = word == 32 && c->tensor_cores;
    const int h = r1.split_h;
    const bool mid = ntt_has_mid(c->log_n);
    info[HEMUL_INFO_WORD] = word;
    info[HEMUL_INFO_NP1] = r1.np;
    info[HEMUL_INFO_NP2] = r2.np;
    info[HEMUL_INFO_SPLIT_H] = h;
    info[HEMUL_INFO_CRT1_TC] = tc && r1.tc_table(0, h) && r1.tc_table(h, log_q - h);
    info[HEMUL_INFO_CRT2_TC] = tc && r2.tc_table(0, log_q);
    info[HEMUL_INFO_BIG_TC] = tc && bs.icrt_tc && bs.fin_tc;
    info[HEMUL_INFO_FUSED_MID] = mid;
    info[HEMUL_INFO_BLK_MONT] = word == 32 && mid && ntt_blk_supported(c->log_n);
    const int tS = ntt_pass_a_levels(c->log_n);
    info[HEMUL_INFO_T_PASS_A] =
        (tc && c->transposed && info[HEMUL_INFO_BIG_TC] && info[HEMUL_INFO_BLK_MONT] &&
         info[HEMUL_INFO_CRT1_TC] && info[HEMUL_INFO_CRT2_TC] &&
         ntt_col_transposed_supported(c->log_n, tS))
            ? tS
            : 0;
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_he_mul_trace(hemul_gpu_ctx* c, int log_q, size_t batch,
                                    const uint64_t* c1_ax, const uint64_t* c1_bx,
                                    const uint64_t* c2_ax, const uint64_t* c2_bx,
                                    const uint64_t* evk_ax, const uint64_t* evk_bx,
                                    uint64_t evk_id, int checkpoint, void* dst, size_t cap,
                                    size_t* written) {
  if (!c || !dst || batch == 0 || checkpoint < HEMUL_TRACE_CRT1 || checkpoint > HEMUL_TRACE_PROD2)
    return HEMUL_E_ARG;
  if (log_q - c->log_p < c->log_p) return fail(c, HEMUL_E_DEPTH, "multiplicative depth exhausted");
  if (!c1_ax || !c1_bx || !c2_ax || !c2_bx) return fail(c, HEMUL_E_ARG, "null buffer");
  return guarded(c, [&]() -> hemul_status {
    Level& lv = get_level(c, log_q);
    const int word = mul_word(c, lv);
    if (evk_ax && evk_bx &&
        (!lv.has_evk || evk_id == 0 || lv.evk_id != evk_id || lv.evk_word != word))
      set_evk_forms(c, lv, evk_ax, evk_bx, evk_id);
    if (!lv.has_evk || lv.evk_word != word)
      return fail(c, HEMUL_E_NO_EVK, "evaluation key not set for this level");
    const size_t poly_w = size_t(c->n) * limbs_of(log_q);
    const size_t out_w = size_t(c->n) * limbs_of(log_q - c->log_p);
    ensure(c->in, 4 * batch * poly_w * 8);
    const uint64_t* src[4] = {c1_ax, c1_bx, c2_ax, c2_bx};
    const uint64_t* in[4];
    for (int t = 0; t < 4; ++t)
      in[t] = stage_in(c, src[t], batch * poly_w, c->in.as<uint64_t>() + t * batch * poly_w);
    ensure(c->outb, 2 * batch * out_w * 8);
    Trace tr;
    tr.stop = checkpoint;
    tr.dst = dst;
    tr.cap = cap;
    ++c->call_id;
    uint64_t* oa = c->outb.as<uint64_t>();
    if (word == 64)
      he_mul_device<F64>(c, lv, log_q, batch, in, oa, oa + batch * out_w, &tr);
    else
      he_mul_device<F32>(c, lv, log_q, batch, in, oa, oa + batch * out_w, &tr);
    if (written) *written = tr.written;
    return HEMUL_OK;
  });
}

}  // extern "C"

// A device-resident ciphertext batch. Its memory comes from the device's
// stream-ordered pool (cudaMallocAsync on the context stream), so creating
// and dropping intermediates inside a chain never synchronises the device.
struct hemul_gpu_ct {
  int device = 0;
  int log_q = 0;
  size_t batch = 0;
  size_t words = 0;  // per polynomial of the batch: n x ceil(log_q / 64)
  uint64_t* mem = nullptr;  // [ax batch | bx batch]
  cudaEvent_t ready = nullptr;  // asynchronous upload still in flight (HEMUL_CT_ASYNC)
  uint64_t* ax() const { return mem; }
  uint64_t* bx() const { return mem + batch * words; }
};

namespace {

struct CtDeleter {
  cudaStream_t st;
  void operator()(hemul_gpu_ct* t) const {
    if (t && t->mem) cudaFreeAsync(t->mem, st);
    if (t && t->ready) cudaEventDestroy(t->ready);
    delete t;
  }
};
using CtPtr = std::unique_ptr<hemul_gpu_ct, CtDeleter>;

CtPtr new_ct(hemul_gpu_ctx* c, int log_q, size_t batch) {
  if (log_q <= 0 || log_q > c->log_q_max) throw std::invalid_argument("log_q out of range");
  if (batch == 0) throw std::invalid_argument("empty ciphertext batch");
  CtPtr t(new hemul_gpu_ct, CtDeleter{c->stream});
  t->device = c->device;
  t->log_q = log_q;
  t->batch = batch;
  t->words = size_t(c->n) * limbs_of(log_q);
  check(cudaMallocAsync(reinterpret_cast<void**>(&t->mem), 2 * batch * t->words * 8, c->stream),
        "ciphertext allocation");
  return t;
}

// Validates a handle and orders the context stream after its upload.
void check_ct(const hemul_gpu_ctx* c, const hemul_gpu_ct* t) {
  if (!t) throw std::invalid_argument("null ciphertext handle");
  if (t->device != c->device) throw std::invalid_argument("ciphertext on another device");
  if (t->words != size_t(c->n) * limbs_of(t->log_q))
    throw std::invalid_argument("ciphertext of another ring degree");
  if (t->ready) check(cudaStreamWaitEvent(c->stream, t->ready, 0), "wait");
}

}  // namespace

extern "C" {

hemul_status hemul_gpu_ct_create(hemul_gpu_ctx* c, int log_q, size_t batch, const uint64_t* ax,
                                 const uint64_t* bx, int flags, hemul_gpu_ct** out) {
  if (!c || !out || (flags & ~HEMUL_CT_ASYNC)) return HEMUL_E_ARG;
  *out = nullptr;
  return guarded(c, [&] {
    auto t = new_ct(c, log_q, batch);
    const size_t bytes = batch * t->words * 8;
    const bool async = flags & HEMUL_CT_ASYNC;
    // async: the copies run on the copy stream (overlapping kernels already
    // queued on the context stream), which waits for the allocation; the
    // context stream then waits for the copies
    cudaStream_t st = async ? c->h2d : c->stream;
    cudaEvent_t ev = nullptr;
    if (async) {
      check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
      check(cudaEventRecord(ev, c->stream), "event");
      check(cudaStreamWaitEvent(c->h2d, ev, 0), "wait");
    }
    for (int s = 0; s < 2; ++s) {
      const uint64_t* src = s ? bx : ax;
      uint64_t* dst = s ? t->bx() : t->ax();
      if (src)
        run_on(c, st, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_H2D, "H2D", [&] {
          return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
        });
      else
        check(cudaMemsetAsync(dst, 0, bytes, st), "ciphertext zero");
    }
    if (async) {
      // the first operation that reads the handle waits for this event
      check(cudaEventRecord(ev, c->h2d), "event");
      t->ready = ev;
    } else {
      // host sources may be reused by the caller as soon as this returns
      check(cudaStreamSynchronize(c->stream), "ciphertext upload");
    }
    *out = t.release();
    return HEMUL_OK;
  });
}

void hemul_gpu_ct_destroy(hemul_gpu_ctx* c, hemul_gpu_ct* t) {
  if (!t) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(t->device);
  if (c && c->device == t->device) {
    if (t->ready) cudaStreamWaitEvent(c->stream, t->ready, 0);  // an upload still in flight
    cudaFreeAsync(t->mem, c->stream);  // after the work queued on the context stream
  } else {
    cudaDeviceSynchronize();
    cudaFree(t->mem);
  }
  if (t->ready) cudaEventDestroy(t->ready);
  delete t;
  cudaSetDevice(cur);
}

hemul_status hemul_gpu_ct_info(const hemul_gpu_ct* t, int* log_q, size_t* batch) {
  if (!t) return HEMUL_E_ARG;
  if (log_q) *log_q = t->log_q;
  if (batch) *batch = t->batch;
  return HEMUL_OK;
}

hemul_status hemul_gpu_ct_device_ptrs(const hemul_gpu_ct* t, uint64_t** ax, uint64_t** bx) {
  if (!t) return HEMUL_E_ARG;
  if (ax) *ax = t->ax();
  if (bx) *bx = t->bx();
  return HEMUL_OK;
}

hemul_status hemul_gpu_ct_download(hemul_gpu_ctx* c, const hemul_gpu_ct* t, uint64_t* ax,
                                   uint64_t* bx) {
  if (!c || !t || !ax || !bx) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check_ct(c, t);
    const size_t bytes = t->batch * t->words * 8;
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H",
        [&] { return cudaMemcpyAsync(ax, t->ax(), bytes, cudaMemcpyDefault, c->stream); });
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H",
        [&] { return cudaMemcpyAsync(bx, t->bx(), bytes, cudaMemcpyDefault, c->stream); });
    check(cudaStreamSynchronize(c->stream), "ciphertext download");
    return HEMUL_OK;
  });
}

}  // extern "C"

namespace {

// Pinned double buffer for file <-> device streaming.
constexpr size_t kPinChunk = size_t(32) << 20;

void ensure_pinned(hemul_gpu_ctx* c) {
  for (int s = 0; s < 2; ++s) {
    if (!c->pinned[s]) check(cudaHostAlloc(&c->pinned[s], kPinChunk, cudaHostAllocDefault), "pinned");
    if (!c->ev_pin[s]) check(cudaEventCreateWithFlags(&c->ev_pin[s], cudaEventDisableTiming), "event");
  }
}

struct File {
  FILE* f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

}  // namespace

extern "C" {

hemul_status hemul_gpu_ct_load(hemul_gpu_ctx* c, const char* path, hemul_gpu_ct** out,
                               int* n_slots) {
  if (!c || !path || !out) return HEMUL_E_ARG;
  *out = nullptr;
  return guarded(c, [&]() -> hemul_status {
    File file;
    file.f = std::fopen(path, "rb");
    if (!file.f) return fail(c, HEMUL_E_IO, std::string("cannot open: ") + path);
    uint32_t h[5];
    if (std::fread(h, 4, 5, file.f) != 5 || std::memcmp(h, "HEA1", 4) != 0)
      return fail(c, HEMUL_E_IO, std::string("bad magic: ") + path);
    if (h[1] != 64) return fail(c, HEMUL_E_ARG, "device ciphertexts use 64-bit words");
    if (h[2] != uint32_t(c->n)) return fail(c, HEMUL_E_ARG, "ciphertext ring degree differs");
    const int log_q = static_cast<int>(h[3]);
    if (log_q <= 0) return fail(c, HEMUL_E_IO, "bad header fields");
    auto t = new_ct(c, log_q, 1);
    ensure_pinned(c);
    // read chunk k into pinned buffer k % 2 while chunk k-1 is copied
    char* dst = reinterpret_cast<char*>(t->mem);
    size_t left = 2 * t->words * 8, off = 0;
    for (int k = 0; left > 0; ++k) {
      const int s = k & 1;
      const size_t sz = std::min(left, kPinChunk);
      check(cudaEventSynchronize(c->ev_pin[s]), "pinned reuse");
      if (std::fread(c->pinned[s], 1, sz, file.f) != sz)
        return fail(c, HEMUL_E_IO, "truncated polynomial data");
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_H2D, "H2D", [&] {
        return cudaMemcpyAsync(dst + off, c->pinned[s], sz, cudaMemcpyHostToDevice, c->stream);
      });
      check(cudaEventRecord(c->ev_pin[s], c->stream), "event");
      off += sz;
      left -= sz;
    }
    check(cudaStreamSynchronize(c->stream), "ciphertext load");
    if (n_slots) *n_slots = static_cast<int>(h[4]);
    *out = t.release();
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_ct_save(hemul_gpu_ctx* c, const hemul_gpu_ct* t, int n_slots,
                               const char* path) {
  if (!c || !t || !path || t->batch != 1) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    check_ct(c, t);
    File file;
    file.f = std::fopen(path, "wb");
    if (!file.f) return fail(c, HEMUL_E_IO, std::string("cannot open for writing: ") + path);
    const uint32_t h[5] = {0, 64, uint32_t(c->n), uint32_t(t->log_q), uint32_t(n_slots)};
    std::fwrite("HEA1", 1, 4, file.f);
    std::fwrite(h + 1, 4, 4, file.f);
    ensure_pinned(c);
    // copy chunk k + 1 while chunk k is written
    const char* src = reinterpret_cast<const char*>(t->mem);
    const size_t total = 2 * t->words * 8;
    const size_t chunks = (total + kPinChunk - 1) / kPinChunk;
    auto issue = [&](size_t k) {
      const size_t off = k * kPinChunk, sz = std::min(kPinChunk, total - off);
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
        return cudaMemcpyAsync(c->pinned[k & 1], src + off, sz, cudaMemcpyDeviceToHost, c->stream);
      });
      check(cudaEventRecord(c->ev_pin[k & 1], c->stream), "event");
    };
    issue(0);
    for (size_t k = 0; k < chunks; ++k) {
      if (k + 1 < chunks) issue(k + 1);
      check(cudaEventSynchronize(c->ev_pin[k & 1]), "ciphertext save");
      const size_t sz = std::min(kPinChunk, total - k * kPinChunk);
      if (std::fwrite(c->pinned[k & 1], 1, sz, file.f) != sz)
        return fail(c, HEMUL_E_IO, std::string("write failed: ") + path);
    }
    if (std::fflush(file.f) != 0) return fail(c, HEMUL_E_IO, std::string("write failed: ") + path);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_ct_he_mul(hemul_gpu_ctx* c, const hemul_gpu_ct* c1, const hemul_gpu_ct* c2,
                                 const uint64_t* evk_ax, const uint64_t* evk_bx, uint64_t evk_id,
                                 hemul_gpu_ct** out) {
  if (!c || !c1 || !c2 || !out) return HEMUL_E_ARG;
  *out = nullptr;
  if (c1->log_q != c2->log_q)
    return fail(c, HEMUL_E_MODULUS_MISMATCH, "ciphertext modulus mismatch");
  const int log_q = c1->log_q;
  if (log_q - c->log_p < c->log_p)
    return fail(c, HEMUL_E_DEPTH, "multiplicative depth exhausted");
  if (c1->batch != c2->batch) return fail(c, HEMUL_E_ARG, "ciphertext batches differ");
  return guarded(c, [&]() -> hemul_status {
    check_ct(c, c1);
    check_ct(c, c2);
    Level& lv = get_level(c, log_q);
    const int word = mul_word(c, lv);
    if (evk_ax && evk_bx &&
        (!lv.has_evk || evk_id == 0 || lv.evk_id != evk_id || lv.evk_word != word))
      set_evk_forms(c, lv, evk_ax, evk_bx, evk_id);
    if (!lv.has_evk || lv.evk_word != word)
      return fail(c, HEMUL_E_NO_EVK, "evaluation key not set for this level");
    auto r = new_ct(c, log_q - c->log_p, c1->batch);
    ++c->call_id;
    const uint64_t* in[4] = {c1->ax(), c1->bx(), c2->ax(), c2->bx()};
    he_mul_any(c, lv, log_q, c1->batch, in, r->ax(), r->bx());
    *out = r.release();  // asynchronous: ordered on the context stream
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_ct_rescale(hemul_gpu_ctx* c, const hemul_gpu_ct* t, hemul_gpu_ct** out) {
  if (!c || !t || !out) return HEMUL_E_ARG;
  *out = nullptr;
  if (t->log_q - c->log_p < c->log_p)
    return fail(c, HEMUL_E_DEPTH, "modulus exhausted; cannot rescale");
  return guarded(c, [&] {
    check_ct(c, t);
    auto r = new_ct(c, t->log_q - c->log_p, t->batch);
    for (int s = 0; s < 2; ++s)
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "rescale", [&] {
        return shift_right(s ? t->bx() : t->ax(), s ? r->bx() : r->ax(), t->batch, c->log_n,
                           t->log_q, c->log_p, c->stream);
      });
    *out = r.release();
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_ct_mod_down(hemul_gpu_ctx* c, const hemul_gpu_ct* t, int new_log_q,
                                   hemul_gpu_ct** out) {
  if (!c || !t || !out) return HEMUL_E_ARG;
  *out = nullptr;
  if (new_log_q <= 0 || new_log_q > t->log_q) return fail(c, HEMUL_E_ARG, "new_log_q out of range");
  return guarded(c, [&] {
    check_ct(c, t);
    auto r = new_ct(c, new_log_q, t->batch);
    for (int s = 0; s < 2; ++s)
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "mod_down", [&] {
        return mod_down(s ? t->bx() : t->ax(), s ? r->bx() : r->ax(), t->batch, c->log_n,
                        t->log_q, new_log_q, c->stream);
      });
    *out = r.release();
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_mul_by_ternary(hemul_gpu_ctx* c, int log_q, size_t batch,
                                      const uint64_t* a, const int32_t* t, uint64_t* out) {
  if (!c || !a || !t || !out || batch == 0) return HEMUL_E_ARG;
  if (log_q <= 0 || log_q > 4 * c->log_q_max) return fail(c, HEMUL_E_ARG, "log_q out of range");
  return guarded(c, [&]() -> hemul_status {
    const int n = c->n, L = limbs_of(log_q);
    // the nonzero coefficients of the ternary polynomial, host side (the
    // caller's vector); nz = 2 i + (t_i < 0)
    std::vector<int> nz;
    for (int i = 0; i < n; ++i) {
      if (t[i] != 0 && t[i] != 1 && t[i] != -1)
        return fail(c, HEMUL_E_ARG, "ternary coefficients must be -1, 0 or 1");
      if (t[i]) nz.push_back(2 * i + (t[i] < 0));
    }
    const size_t words = size_t(n) * L;
    ensure(c->tern_a, 2 * words * 8);
    ensure(c->tern_b, words * 8);
    ensure(c->tern_nz, (nz.size() + 1) * sizeof(int));
    uint64_t* aT = c->tern_a.as<uint64_t>();
    uint64_t* stage = aT + words;
    uint64_t* rT = c->tern_b.as<uint64_t>();
    if (!nz.empty())
      check(cudaMemcpyAsync(c->tern_nz.ptr, nz.data(), nz.size() * sizeof(int),
                            cudaMemcpyHostToDevice, c->stream), "ternary upload");
    for (size_t b = 0; b < batch; ++b) {
      const uint64_t* src = stage_in(c, a + b * words, words, stage);
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "transpose",
          [&] { return word_transpose(src, aT, n, L, c->stream); });
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "mul_by_ternary", [&] {
        return mul_by_ternary(aT, c->tern_nz.as<int>(), static_cast<int>(nz.size()), rT,
                              c->log_n, log_q, c->stream);
      });
      const bool dev = is_device(c, out + b * words);
      uint64_t* dst = dev ? out + b * words : stage;
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "transpose",
          [&] { return word_transpose(rT, dst, L, n, c->stream); });
      if (!dev)
        run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
          return cudaMemcpyAsync(out + b * words, dst, words * 8, cudaMemcpyDefault, c->stream);
        });
    }
    check(cudaStreamSynchronize(c->stream), "mul_by_ternary");
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_rescale(hemul_gpu_ctx* c, int log_q, size_t batch, const uint64_t* ax,
                               const uint64_t* bx, uint64_t* out_ax, uint64_t* out_bx) {
  if (!c) return HEMUL_E_ARG;
  // heaan.cpp:329-330
  if (log_q - c->log_p < c->log_p)
    return fail(c, HEMUL_E_DEPTH, "modulus exhausted; cannot rescale");
  if (batch == 0) return HEMUL_OK;
  if (!ax || !bx || !out_ax || !out_bx) return fail(c, HEMUL_E_ARG, "null buffer");
  return guarded(c, [&]() -> hemul_status {
    const size_t n = size_t(c->n);
    const int L = limbs_of(log_q), Lo = limbs_of(log_q - c->log_p);
    const size_t w = batch * n * L, ow = batch * n * Lo;
    ensure(c->rescale_buf, 2 * w * 8);
    const uint64_t* a = stage_in(c, ax, w, c->rescale_buf.as<uint64_t>());
    const uint64_t* b = stage_in(c, bx, w, c->rescale_buf.as<uint64_t>() + w);
    const OutPair o = out_pair(c, out_ax, out_bx, ow, c->outb);
    for (int t = 0; t < 2; ++t)
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_EPILOGUE, "rescale", [&] {
        return shift_right(t ? b : a, t ? o.b : o.a, batch, c->log_n, log_q, c->log_p,
                           c->stream);
      });
    copy_out(c, o, out_ax, out_bx, ow);
    return HEMUL_OK;
  });
}

}  // extern "C"

namespace {

// One batched HE Mul on device buffers, every launch on c->stream, in the
// prime basis of field F (fields.cuh).
// True when the trace stops here (after copying `bytes` of `src` out).
bool trace_at(hemul_gpu_ctx* c, Trace* tr, int point, const void* src, size_t bytes) {
  if (!tr || tr->stop != point) return false;
  if (bytes > tr->cap) throw std::invalid_argument("trace buffer too small");
  check(cudaMemcpyAsync(tr->dst, src, bytes, cudaMemcpyDefault, c->stream), "trace copy");
  check(cudaStreamSynchronize(c->stream), "trace copy");
  tr->written = bytes;
  return true;
}

template <class F>
void he_mul_device(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                   const uint64_t* const in[4], uint64_t* out_ax, uint64_t* out_bx, Trace* tr) {
  using W = typename F::W;
  const size_t n = size_t(c->n);
  const int log_n = c->log_n;
  const int L = limbs_of(log_q);
  const Basis& bs = get_basis(c, lv, sizeof(W) == 8 ? 64 : 32);
  const RegionDev& r1 = *bs.r1;
  const RegionDev& r2 = *bs.r2;
  const size_t B = batch;
  const size_t poly_w = n * L;
  const typename F::Prime* p1 = r1.P<F>();
  const typename F::Prime* p2 = r2.P<F>();
  // ---- region 1: d0 = bx1 bx2, d1 = ax1 bx2 + ax2 bx1, d2 = ax1 ax2 ---------
  // F64: one RNS operand per input, products d2 (slot 0), d0 (1), d1 (2).
  // F32: every input split at bit h (level_tables.hpp split_h): slots
  // x1 X1 y1 Y1 x2 X2 y2 Y2, products d2 = (0, 1), d0 = (2, 3), d1 = (4, 5)
  // as (c0, c1) with d = c0 + 2^h c1 mod 2^log_q.
  constexpr bool kSplit = sizeof(W) == 4;
  constexpr int kInSlots = kSplit ? 8 : 4, kOutSlots = kSplit ? 6 : 3;
  const int h = r1.split_h;
  const size_t r1w = B * r1.np * n;  // one RNS operand slot
  ensure(c->r1, kInSlots * r1w * sizeof(W));
  W* R1 = c->r1.as<W>();
  const CrtWeights* w1 = r1.weights(kSplit ? h : log_q);
  // int8 tensor-core iCRT + finisher (30-bit split basis): the inverse NTTs
  // feeding them output t_j directly
  bool tc_big = false;
  if constexpr (kSplit) tc_big = c->tensor_cores && bs.icrt_tc && bs.fin_tc;
  const bool mid = ntt_has_mid(log_n);
  // the warp-per-block middle pass (30-bit basis) Montgomery-reduces its
  // products (ntt_blk.cu); the following inverse pass compensates
  const bool blk_mont = kSplit && mid && ntt_blk_supported(log_n);
  // transposed pass-A layout (ntt_col.cu TR forms): both tensor-core CRTs
  // write column-major rows, forward pass A reads them and writes natural
  // rows into a second buffer, the middle pass runs there, inverse pass A
  // writes column-major t rows back for the tensor-core iCRT / finisher
  const int tS = ntt_pass_a_levels(log_n);
  const bool trn = kSplit && c->transposed && c->tensor_cores && tc_big && blk_mont &&
                   ntt_col_transposed_supported(log_n, tS) && r1.tc_table(0, h) &&
                   r1.tc_table(h, log_q - h) && r2.tc_table(0, log_q);
  if constexpr (kSplit) {
    const uint64_t* polys[8];
    int bit0[8], bits[8];
    for (int t = 0; t < 8; ++t) {
      polys[t] = in[t / 2];
      bit0[t] = (t & 1) ? h : 0;
      bits[t] = (t & 1) ? log_q - h : h;
    }
    const CrtTcTable* tlo = c->tensor_cores ? r1.tc_table(0, h) : nullptr;
    const CrtTcTable* thi = c->tensor_cores ? r1.tc_table(h, log_q - h) : nullptr;
    if (tlo && thi) {
      CrtTcTable tabs[8];
      for (int t = 0; t < 8; ++t) tabs[t] = (t & 1) ? *thi : *tlo;
      run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT r1 (tensor cores)", [&] {
        return crt_forward_tc(polys, tabs, 8, L, B, log_n, p1, r1.np, R1, c->stream,
                              trn ? tS : 0);
      });
    } else {
      run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT r1", [&] {
        return crt_forward_multi<F>(polys, 8, L, B, log_n, *w1, p1, r1.np, R1, c->stream, bit0,
                                    bits);
      });
    }
  } else {
    // one launch: ax1 -> A1, bx1 -> B1, ax2 -> A2, bx2 -> B2 (R1 is [A1|B1|A2|B2])
    run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT r1", [&] {
      return crt_forward_multi<F>(in, 4, L, B, log_n, *w1, p1, r1.np, R1, c->stream);
    });
  }
  if (trace_at(c, tr, HEMUL_TRACE_CRT1, R1, kInSlots * r1w * sizeof(W))) return;
  if (trn) {
    if constexpr (kSplit) {
      const int S = tS;
      ensure(c->r1b, kInSlots * r1w * sizeof(W));
      W* R1b = c->r1b.as<W>();
      run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_NTT_A, "NTT pass A (transposed in)", [&] {
        return ntt_col_pass_transposed(false, R1, R1b, kInSlots * B * r1.np, r1.np, log_n, S,
                                       r1.TW<F>(), r1.twc.as<const Twiddle32>(), p1, c->stream);
      });
      run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_MID_R1, "NTT mid r1", [&] {
        return ntt_mid_tensor_split(R1b, B, r1.np, log_n, r1.TW<F>(), r1.ITW<F>(), p1, c->stream);
      });
      run(c, HEMUL_STAGE_INTT, HEMUL_KCLASS_INTT_A, "iNTT pass A (transposed out)", [&] {
        return ntt_col_pass_transposed(true, R1b, R1, kOutSlots * B * r1.np, r1.np, log_n, S,
                                       r1.ITW<F>(), r1.itwc.as<const Twiddle32>(), r1.primes_tm.as<const DevPrime32>(),
                                       c->stream);
      });
    }
  } else if (mid) {
    // forward pass A, then one fused pass: forward pass B + tensor product +
    // inverse pass B, then inverse pass A
    ntt_fwd<F>(c, r1, R1, kInSlots * B * r1.np, HEMUL_STAGE_NTT, 1);
    run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_MID_R1, "NTT mid r1", [&] {
      if constexpr (kSplit)
        return ntt_mid_tensor_split(R1, B, r1.np, log_n, r1.TW<F>(), r1.ITW<F>(), p1, c->stream);
      else  // in place: d2 -> A1, d0 -> B1, d1 -> A2
        return ntt_mid_tensor<F>(R1, R1 + r1w, R1 + 2 * r1w, R1 + 3 * r1w, B, r1.np, log_n,
                                 r1.TW<F>(), r1.ITW<F>(), p1, c->stream);
    });
    ntt_inv<F>(c, r1, R1, kOutSlots * B * r1.np, HEMUL_STAGE_INTT, 1, tc_big, blk_mont);
  } else {
    ntt_fwd<F>(c, r1, R1, kInSlots * B * r1.np, HEMUL_STAGE_NTT);
    // pointwise products are booked under iCRT like rns.cpp:364
    run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_TENSOR, "tensor product", [&] {
      if constexpr (kSplit)
        return tensor_split_product(R1, B, r1.np, log_n, p1, c->stream);
      else
        return tensor_product<F>(R1, R1 + r1w, R1 + 2 * r1w, R1 + 3 * r1w, R1 + r1w,
                                 R1 + 2 * r1w, R1, B, r1.np, log_n, p1, c->stream);
    });
    ntt_inv<F>(c, r1, R1, kOutSlots * B * r1.np, HEMUL_STAGE_INTT, 2, tc_big);
  }
  if (trace_at(c, tr, HEMUL_TRACE_PROD1, R1, kOutSlots * r1w * sizeof(W))) return;
  // d2 = ax1 ax2 mod q in binary (ModUp input); d0 / d1 stay in RNS form
  // and are reconstructed inside the finisher
  ensure(c->dpoly, B * poly_w * 8);
  uint64_t* d2 = c->dpoly.as<uint64_t>();
  bool icrt_done = false;
  if constexpr (kSplit) {
    if (tc_big) {
      const BigTcDev& T = *bs.icrt_tc;
      // t rows: R1 = 8 slots of B x np1 rows; d2 = (slot 0, slot 1)
      alignas(64) CUtensorMap rmap;
      make_raw_tmap(&rmap, R1, n, uint64_t(kInSlots) * B * r1.np);
      const void* rmaps[2] = {&rmap, &rmap};
      BigTcSeg segs[2];
      for (int h2 = 0; h2 < 2; ++h2) {
        segs[h2].row0 = h2 * static_cast<int>(B) * r1.np;
        segs[h2].erows = r1.np;
        segs[h2].primes = p1;
      }
      BigTcOut o;
      o.out0 = o.out1 = d2;
      o.out_limbs = L;
      o.out_bit = T.out_bit;
      o.out_bits = T.out_bits;
      o.tS = trn ? tS : 0;
      run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_ICRT, "iCRT r1 (tensor cores)", [&] {
        return bigint_tc(T.t, segs, static_cast<int>(B), static_cast<int>(B), log_n, o, rmaps,
                         c->stream);
      });
      icrt_done = true;
    }
  }
  if (!icrt_done) {
    run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_ICRT, "iCRT r1", [&] {
      return icrt<F>(R1, B, log_n, p1, r1.np, r1.icrt, d2, c->stream, nullptr,
                     kSplit ? R1 + r1w : nullptr);
    });
  }
  if (trace_at(c, tr, HEMUL_TRACE_D2, d2, B * poly_w * 8)) return;
  const W* D1 = R1 + (kSplit ? 4 : 2) * r1w;  // d1 (c0)
  const W* D0 = R1 + (kSplit ? 2 : 1) * r1w;  // d0 (c0)
  // ---- region 2: ModUp (CRT of d2), evk product, ModDown ------------------
  const size_t r2w = B * r2.np * n;
  ensure(c->r2, 2 * r2w * sizeof(W));
  W* KA = c->r2.as<W>();
  W* KB = KA + r2w;
  bool r2_done = false;
  if constexpr (kSplit) {
    if (const CrtTcTable* t2 = c->tensor_cores ? r2.tc_table(0, log_q) : nullptr) {
      const uint64_t* d2c = d2;
      run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT r2 (tensor cores)", [&] {
        return crt_forward_tc(&d2c, t2, 1, L, B, log_n, p2, r2.np, KA, c->stream,
                              trn ? tS : 0);
      });
      r2_done = true;
    }
  }
  if (!r2_done) {
    run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT r2", [&] {
      return crt_forward<F>(d2, L, B, log_n, *r2.weights(log_q), p2, r2.np, KA, c->stream);
    });
  }
  if (trace_at(c, tr, HEMUL_TRACE_CRT2, KA, r2w * sizeof(W))) return;
  const W* EA = lv.evk_a.as<W>();
  const W* EB = EA + size_t(r2.np) * n;
  if (trn) {
    if constexpr (kSplit) {
      const int S = tS;
      ensure(c->r2b, 2 * r2w * sizeof(W));
      W* Y0 = c->r2b.as<W>();
      W* Y1 = Y0 + r2w;
      run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_NTT_A, "NTT pass A r2 (transposed in)", [&] {
        return ntt_col_pass_transposed(false, KA, Y0, B * r2.np, r2.np, log_n, S, r2.TW<F>(),
                                       r2.twc.as<const Twiddle32>(), p2, c->stream);
      });
      run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_MID_R2, "NTT mid r2", [&] {
        return ntt_mid_evk<F>(Y0, EA, EB, Y0, Y1, B, r2.np, log_n, r2.TW<F>(), r2.ITW<F>(), p2,
                              c->stream);
      });
      run(c, HEMUL_STAGE_INTT, HEMUL_KCLASS_INTT_A, "iNTT pass A r2 (transposed out)", [&] {
        return ntt_col_pass_transposed(true, Y0, KA, 2 * B * r2.np, r2.np, log_n, S, r2.ITW<F>(),
                                       r2.itwc.as<const Twiddle32>(), r2.primes_tm.as<const DevPrime32>(), c->stream);
      });
    }
  } else if (mid) {
    ntt_fwd<F>(c, r2, KA, B * r2.np, HEMUL_STAGE_NTT, 1);
    run(c, HEMUL_STAGE_NTT, HEMUL_KCLASS_MID_R2, "NTT mid r2", [&] {
      return ntt_mid_evk<F>(KA, EA, EB, KA, KB, B, r2.np, log_n, r2.TW<F>(), r2.ITW<F>(), p2,
                            c->stream);
    });
    ntt_inv<F>(c, r2, KA, 2 * B * r2.np, HEMUL_STAGE_INTT, 1, tc_big, blk_mont);
  } else {
    ntt_fwd<F>(c, r2, KA, B * r2.np, HEMUL_STAGE_NTT);
    run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_EVK, "evk product",
        [&] { return evk_product<F>(KA, EA, EB, KA, KB, B, r2.np, log_n, p2, c->stream); });
    ntt_inv<F>(c, r2, KA, 2 * B * r2.np, HEMUL_STAGE_INTT, 2, tc_big);
  }
  if (trace_at(c, tr, HEMUL_TRACE_PROD2, KA, 2 * r2w * sizeof(W))) return;
  // ---- finisher: out = R_logp(d + R_logQ(ks)) for ax (ks_a, d1) and bx
  // (ks_b, d0), exact iCRTs of both regions fused with ModDown + rescale
  IcrtFlags flags;
  flags.capacity = static_cast<unsigned>(2 * B * n);
  ensure(c->flagbuf, (size_t(flags.capacity) + 1) * sizeof(unsigned));
  flags.count = c->flagbuf.as<unsigned>();
  flags.ids = flags.count + 1;
  Finisher fin = bs.fin;
  fin.hi_off = kSplit ? r1w : 0;
  bool fin_done = false;
  if constexpr (kSplit) {
    if (tc_big) {
      const BigTcDev& T = *bs.fin_tc;
      // t rows: map 0 = KA|KB (2B x np2 rows: entries e < B ks_a, e >= B
      // ks_b), map 1 = R1 slots (d1 = slots 4, 5 for ax; d0 = slots 2, 3 for bx)
      alignas(64) CUtensorMap rmap2, rmap1;
      make_raw_tmap(&rmap2, KA, n, 2 * uint64_t(B) * r2.np);
      make_raw_tmap(&rmap1, R1, n, uint64_t(kInSlots) * B * r1.np);
      const void* rmaps[2] = {&rmap2, &rmap1};
      const int Bi = static_cast<int>(B);
      BigTcSeg segs[3];
      segs[0].map = 0;
      segs[0].erows = r2.np;
      segs[0].half_rows = Bi * r2.np;
      segs[0].primes = p2;
      for (int h2 = 0; h2 < 2; ++h2) {  // c0 then c1 (the next slot)
        segs[1 + h2].map = 1;
        segs[1 + h2].row0 = (4 + h2) * Bi * r1.np;
        segs[1 + h2].erows = r1.np;
        segs[1 + h2].half_rows = -2 * Bi * r1.np;
        segs[1 + h2].primes = p1;
      }
      BigTcOut o;
      o.out0 = out_ax;
      o.out1 = out_bx;
      o.out_limbs = limbs_of(log_q - c->log_p);
      o.out_bit = T.out_bit;
      o.out_bits = T.out_bits;
      o.check_amb = 1;
      o.force_exact = c->force_exact;
      o.flags = flags;
      o.tS = trn ? tS : 0;
      run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_FINISH, "finisher (tensor cores)", [&] {
        cudaError_t e = bigint_tc(T.t, segs, static_cast<int>(2 * B), static_cast<int>(B), log_n, o,
                                  rmaps, c->stream);
        if (e != cudaSuccess) return e;
        Finisher ft = fin;
        ft.t_inputs = 1;
        ft.tS = trn ? tS : 0;
        return finish_fixup<F32>(KA, D1, D0, B, log_n, p2, r2.np, p1, r1.np, ft, r2.icrt,
                                 r1.icrt, out_ax, out_bx, flags, c->stream);
      });
      fin_done = true;
    }
  }
  if (!fin_done) {
    run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_FINISH, "finisher", [&] {
      return finish_keyswitch<F>(KA, D1, D0, B, log_n, p2, r2.np, p1, r1.np, fin, r2.icrt,
                                 r1.icrt, out_ax, out_bx, flags, c->force_exact, c->stream);
    });
  }
  ++c->launches;  // the (normally empty) exact fix-up kernel
}

// Row-indexed launches put rows on gridDim.y (<= 65535): a batch is run in
// sub-batches whose largest row count (region-1 operand slots x np1, or the
// 2 np2 region-2 rows) fits.
constexpr size_t kMaxGridY = 65535;

size_t max_sub_batch(const Basis& bs, int word) {
  const size_t per = std::max<size_t>(size_t(word == 64 ? 4 : 8) * bs.r1->np, 2 * size_t(bs.r2->np));
  return std::max<size_t>(1, kMaxGridY / per);
}

void he_mul_any(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                const uint64_t* const in[4], uint64_t* out_ax, uint64_t* out_bx) {
  const int word = lv.evk_word;
  const size_t sub = max_sub_batch(get_basis(c, lv, word), word);
  const size_t poly_w = size_t(c->n) * limbs_of(log_q);
  const size_t out_w = size_t(c->n) * limbs_of(log_q - c->log_p);
  for (size_t b0 = 0; b0 < batch; b0 += sub) {
    const size_t bc = std::min(sub, batch - b0);
    const uint64_t* part[4];
    for (int t = 0; t < 4; ++t) part[t] = in[t] + b0 * poly_w;
    if (word == 64)
      he_mul_device<F64>(c, lv, log_q, bc, part, out_ax + b0 * out_w, out_bx + b0 * out_w);
    else
      he_mul_device<F32>(c, lv, log_q, bc, part, out_ax + b0 * out_w, out_bx + b0 * out_w);
  }
}

// Host buffers: the batch runs in chunks through double-buffered device
// staging so that the H2D copy of chunk k+1 and the D2H copy of chunk k-1
// (two copy streams) overlap the kernels of chunk k (compute stream).
void he_mul_pipelined(hemul_gpu_ctx* c, Level& lv, int log_q, size_t batch,
                      const uint64_t* const src[4], bool dev_in, uint64_t* out_ax,
                      uint64_t* out_bx, bool dev_out) {
  const size_t n = size_t(c->n);
  const size_t poly_w = n * limbs_of(log_q), out_w = n * limbs_of(log_q - c->log_p);
  // 8 chunks: the copies dominate (PCIe moves ~240 MB per HE Mul at X), so
  // small chunks shorten the un-overlapped first H2D and last compute + D2H
  const size_t chunk = batch <= 1 ? 1 : (batch + 7) / 8;
  const size_t chunks = (batch + chunk - 1) / chunk;
  ensure(c->in, 2 * 4 * chunk * poly_w * 8);
  ensure(c->outb, 2 * 2 * chunk * out_w * 8);
  uint64_t* in_slot[2] = {c->in.as<uint64_t>(), c->in.as<uint64_t>() + 4 * chunk * poly_w};
  uint64_t* out_slot[2] = {c->outb.as<uint64_t>(), c->outb.as<uint64_t>() + 2 * chunk * out_w};
  for (size_t k = 0; k < chunks; ++k) {
    const size_t b0 = k * chunk, bc = std::min(chunk, batch - b0);
    const int s = static_cast<int>(k & 1);
    // inputs: wait until chunk k-2 (same slot) finished computing
    if (k >= 2) check(cudaStreamWaitEvent(c->h2d, c->ev_comp[s], 0), "wait");
    const uint64_t* in[4];
    for (int t = 0; t < 4; ++t) {
      if (dev_in) {
        in[t] = src[t] + b0 * poly_w;
      } else {
        uint64_t* d = in_slot[s] + t * chunk * poly_w;
        run_on(c, c->h2d, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_H2D, "H2D", [&] {
          return cudaMemcpyAsync(d, src[t] + b0 * poly_w, bc * poly_w * 8,
                                 cudaMemcpyDefault, c->h2d);
        });
        in[t] = d;
      }
    }
    check(cudaEventRecord(c->ev_h2d[s], c->h2d), "event");
    check(cudaStreamWaitEvent(c->stream, c->ev_h2d[s], 0), "wait");
    // outputs: wait until chunk k-2's results left the slot
    if (k >= 2 && !dev_out) check(cudaStreamWaitEvent(c->stream, c->ev_d2h[s], 0), "wait");
    uint64_t* oa = dev_out ? out_ax + b0 * out_w : out_slot[s];
    uint64_t* ob = dev_out ? out_bx + b0 * out_w : out_slot[s] + chunk * out_w;
    he_mul_any(c, lv, log_q, bc, in, oa, ob);
    check(cudaEventRecord(c->ev_comp[s], c->stream), "event");
    if (!dev_out) {
      check(cudaStreamWaitEvent(c->d2h, c->ev_comp[s], 0), "wait");
      run_on(c, c->d2h, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
        return cudaMemcpyAsync(out_ax + b0 * out_w, oa, bc * out_w * 8, cudaMemcpyDefault,
                               c->d2h);
      });
      run_on(c, c->d2h, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
        return cudaMemcpyAsync(out_bx + b0 * out_w, ob, bc * out_w * 8, cudaMemcpyDefault,
                               c->d2h);
      });
      check(cudaEventRecord(c->ev_d2h[s], c->d2h), "event");
    }
  }
  // the call returns with the results in place (like the synchronous reference)
  check(cudaStreamSynchronize(dev_out ? c->stream : c->d2h), "he_mul");
  check(cudaStreamSynchronize(c->stream), "he_mul");
  // later work on the caller's stream must see the copies done
  if (!dev_out) check(cudaStreamWaitEvent(c->stream, c->ev_d2h[(chunks - 1) & 1], 0), "wait");
}

}  // namespace

extern "C" {

uint64_t hemul_ciphertext_digest(int log_q, size_t words, const uint64_t* ax,
                                 const uint64_t* bx) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&h](uint64_t v) {
    for (int k = 0; k < 8; ++k) h = (h ^ ((v >> (8 * k)) & 0xff)) * 1099511628211ull;
  };
  mix(static_cast<uint64_t>(log_q));
  for (size_t i = 0; i < words; ++i) mix(ax[i]);
  for (size_t i = 0; i < words; ++i) mix(bx[i]);
  return h;
}

// ---- stage entry points ------------------------------------------------------

}  // extern "C"

// ---- stage kernels on one region's device tables -----------------------------
// Shared by the level/region entry points (reference primes of a level) and
// the explicit-prime-set objects (hemul_gpu_rns_*, the lower-level C++ API).
// Every pointer may be host or device memory.

struct hemul_gpu_rns {
  int device = 0;
  int log_n = 0;
  int in_bits = 0;
  bool has_ntt = false;
  RegionDev r;
};

namespace {

void stage_ntt(hemul_gpu_ctx* c, const RegionDev& r, int log_n, uint64_t* data, size_t rows,
               int inverse) {
  const size_t n = size_t(1) << log_n;
  const size_t words = rows * n;
  const bool dev = is_device(c, data);
  uint64_t* d = data;
  if (!dev) {
    ensure(c->r1, words * 8);
    d = c->r1.as<uint64_t>();
    stage_in(c, data, words, d);
  }
  // row r uses prime r % np: chunks are whole multiples of np (gridDim.y)
  const size_t step = std::max<size_t>(1, kMaxGridY / size_t(r.np)) * size_t(r.np);
  for (size_t r0 = 0; r0 < rows; r0 += step) {
    const size_t rc = std::min(step, rows - r0);
    const int total = ntt_num_passes(log_n);
    for (int pass = 0; pass < total; ++pass)
      run(c, inverse ? HEMUL_STAGE_INTT : HEMUL_STAGE_NTT,
          inverse ? HEMUL_KCLASS_INTT_A : HEMUL_KCLASS_NTT_A, inverse ? "iNTT" : "NTT", [&] {
            return inverse ? ntt_inverse_pass<F64>(pass, d + r0 * n, rc, r.np, log_n, r.ITW<F64>(),
                                                   r.P<F64>(), c->stream)
                           : ntt_forward_pass<F64>(pass, d + r0 * n, rc, r.np, log_n, r.TW<F64>(),
                                                   r.P<F64>(), c->stream);
          });
  }
  if (!dev)
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
      return cudaMemcpyAsync(data, d, words * 8, cudaMemcpyDefault, c->stream);
    });
  check(cudaStreamSynchronize(c->stream), "ntt");
}

// The GEMM-tiled CRT / iCRT kernels take 32-coefficient tiles: smaller rings
// run on a zero-padded copy with n = 32 (both maps act per coefficient).
constexpr int kMinTileLogN = 5;

void stage_crt(hemul_gpu_ctx* c, const RegionDev& r, int log_n, int in_bits, size_t batch,
               const uint64_t* poly, uint64_t* rns) {
  const CrtWeights* w = r.weights(in_bits);
  if (!w) throw std::invalid_argument("no CRT table for this input width");
  const int L = limbs_of(in_bits);
  const int ln = std::max(log_n, kMinTileLogN);
  const size_t n = size_t(1) << log_n, nt = size_t(1) << ln;
  ensure(c->in, batch * nt * L * 8);
  const uint64_t* src;
  if (ln != log_n) {
    uint64_t* pad = c->in.as<uint64_t>();
    check(cudaMemsetAsync(pad, 0, batch * nt * L * 8, c->stream), "pad");
    check(cudaMemcpy2DAsync(pad, nt * L * 8, poly, n * L * 8, n * L * 8, batch, cudaMemcpyDefault,
                            c->stream), "pad");
    src = pad;
  } else {
    src = stage_in(c, poly, batch * n * L, c->in.as<uint64_t>());
  }
  const size_t words = batch * r.np * nt;
  const bool dev = ln == log_n && is_device(c, rns);
  uint64_t* dst = rns;
  if (!dev) {
    ensure(c->r1, words * 8);
    dst = c->r1.as<uint64_t>();
  }
  run(c, HEMUL_STAGE_CRT, HEMUL_KCLASS_CRT, "CRT", [&] {
    for (size_t b0 = 0; b0 < batch; b0 += kMaxGridY) {  // batch on gridDim.y
      const size_t bc = std::min(kMaxGridY, batch - b0);
      const cudaError_t e = crt_forward<F64>(src + b0 * nt * L, L, bc, ln, *w, r.P<F64>(), r.np,
                                             dst + b0 * r.np * nt, c->stream);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  });
  if (!dev)
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
      return cudaMemcpy2DAsync(rns, n * 8, dst, nt * 8, n * 8, batch * r.np, cudaMemcpyDefault,
                               c->stream);
    });
  check(cudaStreamSynchronize(c->stream), "crt");
}

void stage_pointwise(hemul_gpu_ctx* c, const RegionDev& r, int log_n, size_t batch,
                     const uint64_t* a, const uint64_t* b, uint64_t* out) {
  const size_t words = batch * r.np * (size_t(1) << log_n);
  ensure(c->r1, 3 * words * 8);
  const uint64_t* da = stage_in(c, a, words, c->r1.as<uint64_t>());
  const uint64_t* db = stage_in(c, b, words, c->r1.as<uint64_t>() + words);
  const bool dev = is_device(c, out);
  uint64_t* d = dev ? out : c->r1.as<uint64_t>() + 2 * words;
  run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_TENSOR, "pointwise", [&] {
    return pointwise(da, db, d, batch, r.np, log_n, r.primes.as<DevPrime>(), c->stream);
  });
  if (!dev)
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
      return cudaMemcpyAsync(out, d, words * 8, cudaMemcpyDefault, c->stream);
    });
  check(cudaStreamSynchronize(c->stream), "pointwise");
}

void stage_icrt(hemul_gpu_ctx* c, const RegionDev& r, int log_n, size_t batch, const uint64_t* rns,
                uint64_t* poly) {
  const int ln = std::max(log_n, kMinTileLogN);
  const size_t n = size_t(1) << log_n, nt = size_t(1) << ln;
  const size_t words = batch * r.np * nt;
  const int TL = limbs_of(r.target_bits);
  ensure(c->r1, words * 8);
  const uint64_t* src;
  if (ln != log_n) {
    uint64_t* pad = c->r1.as<uint64_t>();
    check(cudaMemsetAsync(pad, 0, words * 8, c->stream), "pad");
    check(cudaMemcpy2DAsync(pad, nt * 8, rns, n * 8, n * 8, batch * r.np, cudaMemcpyDefault,
                            c->stream), "pad");
    src = pad;
  } else {
    src = stage_in(c, rns, words, c->r1.as<uint64_t>());
  }
  const bool dev = ln == log_n && is_device(c, poly);
  uint64_t* dst = poly;
  if (!dev) {
    ensure(c->ks, batch * nt * TL * 8);
    dst = c->ks.as<uint64_t>();
  }
  // arbitrary residues: the exact fix-up handles |v| >= P/4
  IcrtFlags flags;
  flags.capacity = static_cast<unsigned>(std::min(batch, kMaxGridY) * nt);
  ensure(c->flagbuf, (size_t(flags.capacity) + 1) * sizeof(unsigned));
  flags.count = c->flagbuf.as<unsigned>();
  flags.ids = flags.count + 1;
  run(c, HEMUL_STAGE_ICRT, HEMUL_KCLASS_ICRT, "iCRT", [&] {
    for (size_t b0 = 0; b0 < batch; b0 += kMaxGridY) {  // batch on gridDim.y
      const size_t bc = std::min(kMaxGridY, batch - b0);
      const cudaError_t e = icrt<F64>(src + b0 * r.np * nt, bc, ln, r.P<F64>(), r.np, r.icrt,
                                      dst + b0 * nt * TL, c->stream, &flags);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  });
  ++c->launches;  // the fix-up kernel
  if (!dev)
    run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H", [&] {
      return cudaMemcpy2DAsync(poly, n * TL * 8, dst, nt * TL * 8, n * TL * 8, batch,
                               cudaMemcpyDefault, c->stream);
    });
  check(cudaStreamSynchronize(c->stream), "icrt");
}

const RegionDev& stage_region(hemul_gpu_ctx* c, int log_q, int region) {
  Level& lv = get_level(c, log_q);
  const Basis& bs = get_basis(c, lv, 64);  // stage entry points: reference primes
  return region == 1 ? *bs.r1 : *bs.r2;
}

void check_rns(const hemul_gpu_ctx* c, const hemul_gpu_rns* t) {
  if (!t) throw std::invalid_argument("null prime-set handle");
  if (t->device != c->device) throw std::invalid_argument("prime set on another device");
}

}  // namespace

extern "C" {

hemul_status hemul_gpu_ntt(hemul_gpu_ctx* c, int log_q, int region, uint64_t* data, size_t rows,
                           int inverse) {
  if (!c || !data || (region != 1 && region != 2)) return HEMUL_E_ARG;
  return guarded(c, [&] {
    stage_ntt(c, stage_region(c, log_q, region), c->log_n, data, rows, inverse);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_ntt32(hemul_gpu_ctx* c, int log_q, int region, int np, uint32_t* data,
                             size_t rows, int inverse) {
  if (!c || !data || (region != 1 && region != 2) || np < 0) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    Level& lv = get_level(c, log_q);
    const Basis& bs = get_basis(c, lv, 32);
    const RegionDev& r = region == 1 ? *bs.r1 : *bs.r2;
    if (r.word != 32) return fail(c, HEMUL_E_ARG, "level has no 30-bit basis");
    if (np > r.np) return fail(c, HEMUL_E_ARG, "more primes than the level's basis holds");
    const int npu = np ? np : r.np;  // rows use the first npu primes
    const size_t n = size_t(1) << c->log_n, words = rows * n;
    uint32_t* d = data;
    const bool dev = is_device(c, data);
    if (!dev) {
      ensure(c->r1, words * 4);
      d = c->r1.as<uint32_t>();
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_H2D, "H2D",
          [&] { return cudaMemcpyAsync(d, data, words * 4, cudaMemcpyDefault, c->stream); });
    }
    // row r uses prime r % npu; chunks are whole multiples of npu (gridDim.y)
    const size_t step = std::max<size_t>(1, kMaxGridY / size_t(npu)) * size_t(npu);
    const int total = ntt_num_passes(c->log_n);
    for (size_t r0 = 0; r0 < rows; r0 += step) {
      const size_t rc = std::min(step, rows - r0);
      for (int pass = 0; pass < total; ++pass) {
        const bool a = inverse ? pass + 1 == total : pass == 0;
        run(c, inverse ? HEMUL_STAGE_INTT : HEMUL_STAGE_NTT,
            inverse ? (a ? HEMUL_KCLASS_INTT_A : HEMUL_KCLASS_INTT_B)
                    : (a ? HEMUL_KCLASS_NTT_A : HEMUL_KCLASS_NTT_B),
            inverse ? "iNTT" : "NTT", [&] {
              return inverse ? ntt_inverse_pass<F32>(pass, d + r0 * n, rc, npu, c->log_n,
                                                     r.ITW<F32>(), r.P<F32>(), c->stream)
                             : ntt_forward_pass<F32>(pass, d + r0 * n, rc, npu, c->log_n,
                                                     r.TW<F32>(), r.P<F32>(), c->stream);
            });
      }
    }
    if (!dev)
      run(c, HEMUL_STAGE_EXTRA, HEMUL_KCLASS_D2H, "D2H",
          [&] { return cudaMemcpyAsync(data, d, words * 4, cudaMemcpyDefault, c->stream); });
    check(cudaStreamSynchronize(c->stream), "ntt32");
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_level_twiddles32(hemul_gpu_ctx* c, int log_q, int region, int j,
                                        uint32_t* tw, uint32_t* itw) {
  if (!c || (region != 1 && region != 2) || j < 0) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    Level& lv = get_level(c, log_q);
    const RegionDev& r = region == 1 ? *get_basis(c, lv, 32).r1 : *get_basis(c, lv, 32).r2;
    if (r.word != 32 || j >= r.np) return fail(c, HEMUL_E_ARG, "no such 30-bit basis prime");
    const size_t n = size_t(1) << c->log_n, off = size_t(j) * n;
    if (tw)
      check(cudaMemcpyAsync(tw, r.tw.as<Twiddle32>() + off, n * sizeof(Twiddle32),
                            cudaMemcpyDefault, c->stream), "twiddles");
    if (itw)
      check(cudaMemcpyAsync(itw, r.itw.as<Twiddle32>() + off, n * sizeof(Twiddle32),
                            cudaMemcpyDefault, c->stream), "twiddles");
    check(cudaStreamSynchronize(c->stream), "twiddles");
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_crt(hemul_gpu_ctx* c, int log_q, int region, int in_bits, size_t batch,
                           const uint64_t* poly, uint64_t* rns) {
  if (!c || !poly || !rns || (region != 1 && region != 2)) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    const RegionDev& r = stage_region(c, log_q, region);
    if (!r.weights(in_bits)) return fail(c, HEMUL_E_ARG, "no CRT table for this input width");
    stage_crt(c, r, c->log_n, in_bits, batch, poly, rns);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_pointwise(hemul_gpu_ctx* c, int log_q, int region, size_t batch,
                                 const uint64_t* a, const uint64_t* b, uint64_t* out) {
  if (!c || !a || !b || !out || (region != 1 && region != 2)) return HEMUL_E_ARG;
  return guarded(c, [&] {
    stage_pointwise(c, stage_region(c, log_q, region), c->log_n, batch, a, b, out);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_icrt(hemul_gpu_ctx* c, int log_q, int region, size_t batch,
                            const uint64_t* rns, uint64_t* poly) {
  if (!c || !rns || !poly || (region != 1 && region != 2)) return HEMUL_E_ARG;
  return guarded(c, [&] {
    stage_icrt(c, stage_region(c, log_q, region), c->log_n, batch, rns, poly);
    return HEMUL_OK;
  });
}

// ---- explicit prime sets (the reference's lower-level API) -------------------

hemul_status hemul_gpu_rns_create(hemul_gpu_ctx* c, int log_n, const uint64_t* primes,
                                  const uint64_t* roots, int np, int in_bits, int target_bits,
                                  hemul_gpu_rns** out) {
  if (!c || !out || !primes || np <= 0) return HEMUL_E_ARG;
  *out = nullptr;
  if (log_n < 1 || log_n > 17) return fail(c, HEMUL_E_ARG, "log_n out of range (1..17)");
  if (in_bits < 0 || target_bits < 0) return fail(c, HEMUL_E_ARG, "negative bit width");
  return guarded(c, [&] {
    const std::vector<uint64_t> ps(primes, primes + np);
    const std::vector<uint64_t> rs = roots ? std::vector<uint64_t>(roots, roots + np)
                                           : std::vector<uint64_t>{};
    std::vector<int> crt_bits;
    if (in_bits > 0) crt_bits.push_back(in_bits);
    const RegionHost h = build_explicit_region(ps, rs, log_n, target_bits > 0 ? target_bits : 64,
                                               crt_bits, host_threads());
    auto t = std::make_unique<hemul_gpu_rns>();
    t->device = c->device;
    t->log_n = log_n;
    t->in_bits = in_bits;
    t->has_ntt = roots != nullptr;
    fill_region(t->r, h, c->stream);
    if (target_bits == 0) t->r.target_bits = 0;
    check(cudaStreamSynchronize(c->stream), "prime-set upload");
    *out = t.release();
    return HEMUL_OK;
  });
}

void hemul_gpu_rns_destroy(hemul_gpu_rns* t) {
  if (!t) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(t->device);
  delete t;
  cudaSetDevice(cur);
}

hemul_status hemul_gpu_rns_ntt(hemul_gpu_ctx* c, const hemul_gpu_rns* t, uint64_t* data,
                               size_t rows, int inverse) {
  if (!c || !data) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    check_rns(c, t);
    if (!t->has_ntt) return fail(c, HEMUL_E_ARG, "prime set built without roots (no NTT tables)");
    stage_ntt(c, t->r, t->log_n, data, rows, inverse);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_rns_crt(hemul_gpu_ctx* c, const hemul_gpu_rns* t, size_t batch,
                               const uint64_t* poly, uint64_t* rns) {
  if (!c || !poly || !rns) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    check_rns(c, t);
    if (t->in_bits <= 0) return fail(c, HEMUL_E_ARG, "prime set built without CRT tables");
    stage_crt(c, t->r, t->log_n, t->in_bits, batch, poly, rns);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_rns_pointwise(hemul_gpu_ctx* c, const hemul_gpu_rns* t, size_t batch,
                                     const uint64_t* a, const uint64_t* b, uint64_t* out) {
  if (!c || !a || !b || !out) return HEMUL_E_ARG;
  return guarded(c, [&] {
    check_rns(c, t);
    stage_pointwise(c, t->r, t->log_n, batch, a, b, out);
    return HEMUL_OK;
  });
}

hemul_status hemul_gpu_rns_icrt(hemul_gpu_ctx* c, const hemul_gpu_rns* t, size_t batch,
                                const uint64_t* rns, uint64_t* poly) {
  if (!c || !rns || !poly) return HEMUL_E_ARG;
  return guarded(c, [&]() -> hemul_status {
    check_rns(c, t);
    if (t->r.target_bits <= 0) return fail(c, HEMUL_E_ARG, "prime set built without iCRT tables");
    stage_icrt(c, t->r, t->log_n, batch, rns, poly);
    return HEMUL_OK;
  });
}

}  // extern "C"
