// Host-side construction of one level's tables (the B200 counterpart of
// Scheme::Level, proj/core/src/heaan.cpp:104-112,119-150).
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "device_tables.cuh"

namespace hemul_gpu {

// params.cpp:76-87
int prime_count(int bound_bits, int log_n);
// params.cpp:89-115 (w64): primes p = 1 mod 2n descending from 2^60, their
// smallest-c primitive 2n-th roots. Throws std::runtime_error when exhausted.
void generate_primes(int count, int log_n, std::vector<uint64_t>& primes,
                     std::vector<uint64_t>& roots);
// The B200 basis (fields.cuh F32): the same rule below 2^30.
constexpr int kPrime30Bits = 30;
// Thrown (only) when the 30-bit basis cannot cover a ring degree / level;
// the context then computes in the w64 basis. Every other failure (CUDA,
// allocation, upload) propagates.
struct BasisUnavailable : std::runtime_error {
  using std::runtime_error::runtime_error;
};
void generate_primes30(int count, int log_n, std::vector<uint64_t>& primes,
                       std::vector<uint64_t>& roots);
// iCRT headroom every he_mul region keeps (icrt.cu: fp64 quotient argument)
constexpr int kMinSlackBits = 4;

// The reference's prime set of one region at modulus log_q (w64 rule with the
// grow-until-bound loop of heaan.cpp:132-143), host arithmetic only: no
// twiddle or CRT tables are built. p_limbs = 64-bit limbs of P = prod p_j
// (the PLimbs of the reference's iCRT, params.cpp:215-239).
std::vector<uint64_t> reference_primes(int region, int log_q, int log_q_max, int log_n,
                                       int* p_limbs);

struct RegionHost {
  int region = 0;
  int word = 64;  // 64: reference w64 primes (F64), 32: 30-bit basis (F32)
  int split_h = 0;  // region 1 split into h-bit halves (0: unsplit)
  int np = 0;
  int log_n = 0;
  int target_bits = 0;  // log_q (region 1) or log_q + log_Q (region 2)
  int slack_bits = 0;   // log2(P) - log2(2 * max|v|), the iCRT headroom
  std::vector<uint64_t> primes, roots;
  std::vector<DevPrime> dev;         // np (word 64)
  std::vector<Twiddle> tw, itw;      // np * n each, ShoupPair tables (word 64)
  std::vector<DevPrime32> dev32;     // np (word 32)
  // word 32: the same with ninv, w1n pre-multiplied by (P/p_j)^-1, so that
  // the last inverse-NTT level outputs t_j = x_j (P/p_j)^-1 directly (the
  // operand of the tensor-core iCRT / finisher, bigint_tc.cu)
  std::vector<DevPrime32> dev32_t;
  // word 32: dev32 / dev32_t with ninv, w1n also multiplied by 2^32, for the
  // inverse passes that follow the warp-per-block middle pass, whose
  // evaluation-domain products are Montgomery-reduced (x y 2^-32, ntt_blk.cu)
  std::vector<DevPrime32> dev32_m, dev32_tm;
  // word 32: no host twiddle tables; the device builds them from primes,
  // roots and roots_inv = psi_j^-1 (tables.cu build_twiddles32)
  std::vector<uint64_t> roots_inv;
  // CRT weights per input width (see kernels.hpp CrtWeights)
  struct Crt {
    int in_bits = 0, chunks = 0, ld = 0;
    std::vector<uint32_t> wtab;
  };
  std::vector<Crt> crt;
  // int8 tensor-core CRT tables (word 32; kernels.hpp CrtTcTable), one per
  // input field [bit0, bit0 + bits)
  struct CrtTc {
    int bit0 = 0, bits = 0;
    int kpad = 0, col_tile = 0, ncol_tiles = 0, primes_per_tile = 0, limb0 = 0, end_bit = 0;
    std::vector<uint8_t> btab;
  };
  std::vector<CrtTc> crt_tc;
  // iCRT operands mod 2^T, rows in A order: H_j[, H_j 2^30], ..., (-P)
  // (split: then the same rows times 2^h)
  std::vector<std::vector<uint64_t>> hat_t;
  // iCRT table (see kernels.hpp IcrtTable): hat_t rows in 25-bit chunks
  int m_out = 0, m_pad = 0;
  std::vector<uint32_t> btab;
  // exact iCRT fallback: H_j = P / p_j rows, P, floor(P / 2), p_limbs each
  int p_limbs = 0;
  std::vector<uint64_t> hat_full, big_p, half_p;
};

// Region 1 at modulus log_q: products mod 2^log_q (heaan.cpp:132-138).
// Region 2: key switching, prime product >= 2^(log_q + 2 log_Q + log_n + 1),
// target 2^(log_q + log_Q) (heaan.cpp:139-147). crt_bits lists the input
// widths the region must convert (log_q; region 2 also 2 log_Q for the evk).
// threads > 1 parallelises the twiddle tables. word 64: the reference's
// primes and prime count; word 32: the fewest 30-bit primes with
// kMinSlackBits of iCRT headroom.
// split_h > 0 (region 1): the operands are cut at bit h (h >= log_q / 2),
// a = a0 + 2^h a1, so a b mod 2^log_q = c0 + 2^h c1 with c0 = a0 b0 and
// c1 = a0 b1 + a1 b0 (2^(2h) = 0 mod 2^log_q); the basis only has to hold
// h-bit x h-bit products, the CRT table converts h-bit halves, and the iCRT
// table has the rows of c0 followed by the rows of c1 shifted by h.
RegionHost build_region(int region, int log_q, int log_q_max, int log_n,
                        const std::vector<int>& crt_bits, int threads, int word = 64,
                        int split_h = 0);

// Tables of an explicit w64 prime set (the reference's lower-level API:
// generate_primes / make_crt_tables / make_ntt_tables / make_icrt_tables,
// params.cpp:89-239): twiddles from the given roots, CRT weights per input
// width, iCRT to 2^target_bits. No headroom requirement: the stage iCRT runs
// with the exact fix-up for arbitrary residues.
RegionHost build_explicit_region(const std::vector<uint64_t>& primes,
                                 const std::vector<uint64_t>& roots, int log_n, int target_bits,
                                 const std::vector<int>& crt_bits, int threads);

// Tensor-core CRT table of field [bit0, bit0 + bits) (bit0 % 8 == 0) for the
// region's primes: column tiling chosen so that the weight tile and two
// 128-coefficient A stages fit in shared memory (crt_tc.cu).
// kpad_min: pad K at least this far (fields converted in one launch share
// one K padding and column tiling).
int build_crt_tc_kpad(int bit0, int bits);
RegionHost::CrtTc build_crt_tc(const std::vector<uint64_t>& primes, int bit0, int bits,
                               int kpad_min = 0);
// Split point of the 30-bit basis' region 1: ceil(log_q / 2) rounded up to a
// byte (the tensor-core CRT reads whole bytes), or ceil(log_q / 2) when that
// leaves no high half.
inline int split_point(int log_q) {
  const int h = (log_q + 1) / 2, h8 = (h + 7) / 8 * 8;
  return h8 < log_q ? h8 : h;
}

// Chunk width of the iCRT GEMM's B operand (products 30 x 25 bits, see
// igemm.cuh) and the fraction window kept below bit log_Q by the fused
// key-switch finisher.
constexpr int kChunkBits = 25;
constexpr int kFinisherGuardBits = 125;

// CRT weight-table columns (2 np) padded for crt.cu's tiling: a multiple of
// 16 up to 192 columns (one tile of <= 12 warps), else a multiple of 128
// (tiles of 8 warps).
inline int crt_cols_pad(int cols) {
  const int c16 = (cols + 15) / 16 * 16;
  return c16 <= 192 ? c16 : (cols + 127) / 128 * 128;
}

// Constant operand of the tensor-core iCRT / finisher GEMM (kernels.hpp
// BigTcTable): segments of rows V (< 2^T) with their k rows (-P), the window
// starting at bit base8 (multiple of 8).
struct BigTcHost {
  int n_cols = 0, k_bytes = 0, k_slot = 0, nseg = 0, base8 = 0;
  int slot0[3] = {0, 0, 0}, np[3] = {0, 0, 0};
  // output window (relative to base8); rounding constants are a table row
  int out_bit = 0, out_bits = 0;
  std::vector<uint8_t> btab;  // [k_bytes / 64][n_cols][64] (64-byte swizzled)
};
// iCRT of a split region 1 (d = c0 + 2^h c1 mod 2^log_q, exact from bit 0).
BigTcHost build_icrt_tc(const RegionHost& r1);
// Fused ModDown + add + rescale (same window as build_finisher).
BigTcHost build_finisher_tc(const RegionHost& r1, const RegionHost& r2, int log_q, int log_q_max,
                            int log_p);

// Table of the fused ModDown + add + rescale kernel (kernels.hpp Finisher).
struct FinisherHost {
  int base = 0, width = 0, cols = 0, cols_pad = 0, k2 = 0, k1 = 0;
  int half_q_bit = 0, half_p_bit = 0, out_bit = 0, out_bits = 0;
  std::vector<uint32_t> btab;  // (k2 + k1) x cols_pad
};
FinisherHost build_finisher(const RegionHost& r1, const RegionHost& r2, int log_q, int log_q_max,
                            int log_p);

}  // namespace hemul_gpu
