// Host-callable launchers of the sm_100a kernels (one .cu file per stage).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device_tables.cuh"
#include "fields.cuh"

namespace hemul_gpu {

// Opt-in dynamic shared memory cap we request (227 KB per CTA minus room for
// static shared arrays).
constexpr int kMaxDynSmem = 224 * 1024;

// ---- NTT (ntt.cu) ----------------------------------------------------------
// Every RNS kernel is instantiated for both residue fields (fields.cuh):
// F64 (the reference's w64 primes) and F32 (the B200 30-bit basis).
cudaError_t ntt_setup_attributes();
// rows = batch * np prime-major rows; row r uses prime r % np. One memory
// pass per call: forward pass 0 = levels [0, s1) on columns, pass 1 = levels
// [s1, logN) on blocks; inverse pass 0 = levels [s1, logN), pass 1 = levels
// [0, s1) + n^-1. Outputs of a full transform are canonical.
int ntt_num_passes(int log_n);
int ntt_pass_a_levels(int log_n);  // S of pass A (split_levels s1)
template <class F>
cudaError_t ntt_forward_pass(int pass, typename F::W* data, size_t rows, int np, int log_n,
                             const typename F::Tw* tw, const typename F::Prime* primes,
                             cudaStream_t st);
template <class F>
cudaError_t ntt_inverse_pass(int pass, typename F::W* data, size_t rows, int np, int log_n,
                             const typename F::Tw* itw, const typename F::Prime* primes,
                             cudaStream_t st);

// 30-bit basis pass A (strided levels [0, S), ntt_col.cu): one warp per
// column, shuffles for the lane levels; used by ntt_forward_pass /
// ntt_inverse_pass when supported (S = 6..9, >= 16 columns).
// tables.cu: the 30-bit basis' twiddle tables (make_ntt_tables,
// params.cpp:151-180) on the device; roots_inv = psi_j^-1
cudaError_t build_twiddles32(const uint32_t* primes, const uint32_t* roots,
                             const uint32_t* roots_inv, int np, int log_n, Twiddle32* tw,
                             Twiddle32* itw, cudaStream_t st);
bool ntt_col_supported(int log_n, int S);
// Transposed forms of the column pass (S = 8, 9; out of place): forward reads
// rows in the column-major layout (column x of a row at [x 2^S, (x+1) 2^S))
// and writes the natural layout; inverse reads natural and writes transposed.
bool ntt_col_transposed_supported(int log_n, int S);
// twc (forward): the forward twiddles in the kernel's shared-slot order, per
// prime 2^S pairs (ntt_col_slot_twiddles, built once per level)
cudaError_t ntt_col_pass_transposed(bool inv, const uint32_t* in, uint32_t* out, size_t rows,
                                    int np, int log_n, int S, const Twiddle32* tw,
                                    const Twiddle32* twc, const DevPrime32* primes,
                                    cudaStream_t st);
cudaError_t ntt_col_slot_twiddles(const Twiddle32* tw, int np, int log_n, int S, Twiddle32* out,
                                  cudaStream_t st);
cudaError_t ntt_col_pass(bool inv, uint32_t* data, size_t rows, int np, int log_n, int S,
                         const Twiddle32* tw, const DevPrime32* primes, cudaStream_t st);

// 30-bit basis fused middle pass with one warp per contiguous block
// (ntt_blk.cu); used by ntt_mid_tensor_split / ntt_mid_evk when supported.
bool ntt_blk_supported(int log_n);
cudaError_t ntt_blk_tensor_split(uint32_t* R1, size_t batch, int np, int log_n,
                                 const Twiddle32* tw, const Twiddle32* itw,
                                 const DevPrime32* primes, cudaStream_t st);
cudaError_t ntt_blk_evk(uint32_t* Fin, const uint32_t* ea, const uint32_t* eb, uint32_t* KA,
                        uint32_t* KB, size_t batch, int np, int log_n, const Twiddle32* tw,
                        const Twiddle32* itw, const DevPrime32* primes, cudaStream_t st);

// Fused middle pass (two-pass sizes, logN 12..17): forward levels
// [s1, logN) of every operand + the evaluation-domain product + inverse
// levels [s1, logN) of the products, one read and one write per block.
// Inputs come out of forward pass 0, outputs go into inverse pass 1.
bool ntt_has_mid(int log_n);
// Region 1: A1 B1 A2 B2 -> d2 (over A1), d0 (over B1), d1 = A1B2 + A2B1 (over A2).
template <class F>
cudaError_t ntt_mid_tensor(typename F::W* A1, typename F::W* B1, typename F::W* A2,
                           typename F::W* B2, size_t batch, int np, int log_n,
                           const typename F::Tw* tw, const typename F::Tw* itw,
                           const typename F::Prime* primes, cudaStream_t st);
// Split region 1 (F32::tensor_split): R1 = 8 slots of batch x np x n (the
// halves x1 X1 y1 Y1 x2 X2 y2 Y2); the six half products land in slots 0..5.
cudaError_t ntt_mid_tensor_split(uint32_t* R1, size_t batch, int np, int log_n,
                                 const Twiddle32* tw, const Twiddle32* itw,
                                 const DevPrime32* primes, cudaStream_t st);
// Region 2: F -> F evk_a (KA), F evk_b (KB); KA may alias F.
template <class F>
cudaError_t ntt_mid_evk(typename F::W* Fin, const typename F::W* ea, const typename F::W* eb,
                        typename F::W* KA, typename F::W* KB, size_t batch, int np, int log_n,
                        const typename F::Tw* tw, const typename F::Tw* itw,
                        const typename F::Prime* primes, cudaStream_t st);

// ---- integer-pipe peak probe (probe.cu) ------------------------------------
// Measured IMAD.WIDE.U32 throughput of this device in ops/s (a dependent-free
// stream of mad.wide.u32, 148 x 8 CTAs), and the SM clock it ran at (kHz).
cudaError_t imad_peak(double* ops_per_s, cudaStream_t st);
// Dense int8 tensor-core ops/s (2 per u8 MAC) of tcgen05.mma kind::i8 on this device.
cudaError_t tc_peak(double* ops_per_s, cudaStream_t st);

// ---- CRT (crt.cu) ----------------------------------------------------------
// Weight table for one (prime set, input width), m < chunks = ceil(in_bits /
// 25) (the input is cut into 25-bit chunks: the iGEMM operand widths).
// F64: wtab[m * ld + 2 j + h] = 30-bit half h of 2^(25 m) mod p_j;
// F32: wtab[m * ld + j] = 2^(25 m) mod p_j (< 2^30).
struct CrtWeights {
  const uint32_t* wtab = nullptr;
  int chunks = 0;
  int ld = 0;  // crt_cols_pad(np * F::kCrtColsPerPrime)
};
constexpr int kCrtPrimesPerTile = 16;
constexpr int kMaxCrtInputs = 8;  // inputs of one multi-input CRT launch
cudaError_t crt_setup_attributes();
// poly: batch x n x limbs; out: batch x np x n canonical residues.
template <class F>
cudaError_t crt_forward(const uint64_t* poly, int limbs, size_t batch, int log_n,
                        const CrtWeights& w, const typename F::Prime* primes, int np,
                        typename F::W* out, cudaStream_t st);
// Up to 8 independent inputs of `batch` polys each in one launch; input t
// lands at out + t * batch * np * n and converts bits [bit0[t], bit0[t] +
// bits[t]) of its coefficients (null arrays: bit 0, the table's width).
template <class F>
cudaError_t crt_forward_multi(const uint64_t* const* polys, int count, int limbs, size_t batch,
                              int log_n, const CrtWeights& w, const typename F::Prime* primes,
                              int np, typename F::W* out, cudaStream_t st,
                              const int* bit0 = nullptr, const int* bits = nullptr);

// ---- CRT on the int8 tensor cores (crt_tc.cu, 30-bit basis only) ----------
// One input field: bits [bit0, bit0 + bits) of each coefficient, bit0 % 8 = 0.
// The GEMM reads kpad bytes per coefficient starting at limb limb0 (byte
// offset d = bit0 / 8 - 8 limb0 inside it); bits >= end_bit (= bit0 + bits,
// relative to the coefficient) are cleared on load.
// btab: [ncol_tiles * col_tile][kpad] u8, row 4 jj + b of column tile ct =
// byte b of 2^(8 (k - d) + 32) mod p_j (Montgomery), j = ct * primes_per_tile + jj, for
// d <= k < d + ceil(bits / 8), else 0 (level_tables.cpp build_crt_tc).
struct CrtTcTable {
  const uint8_t* btab = nullptr;
  int kpad = 0;             // multiple of 32
  int col_tile = 0;         // multiple of 16, <= 256 (4 x primes_per_tile, padded)
  int ncol_tiles = 0;
  int primes_per_tile = 0;
  int limb0 = 0;
  int end_bit = 0;
};
cudaError_t crt_tc_setup_attributes();
bool crt_tc_supported(const CrtTcTable& tab);
// Up to 8 inputs (same layout and column tiling, own tables); input t lands
// at out + t * batch * np * n as canonical residues (crt_forward_multi).
cudaError_t crt_forward_tc(const uint64_t* const* polys, const CrtTcTable* tabs, int count,
                           int limbs, size_t batch, int log_n, const DevPrime32* primes, int np,
                           uint32_t* out, cudaStream_t st, int transposed_S = 0);

// ---- iCRT (icrt.cu) --------------------------------------------------------
// B table for the exact reconstruction mod 2^T: (R np + 1) rows x m_pad
// columns of 25-bit chunks, R = F::kRowsPerPrime (F64 rows 2j: H_j mod 2^T,
// 2j+1: H_j 2^30 mod 2^T; F32 row j: H_j mod 2^T; last row (-P) mod 2^T),
// m_out = ceil(T / 25) real columns.
struct IcrtTable {
  const uint32_t* btab = nullptr;
  int m_out = 0;
  int m_pad = 0;  // multiple of 16
  int target_bits = 0;
  // exact fallback (arbitrary residues): H_j = P/p_j, P, floor(P/2), each
  // p_limbs words (H_j rows back to back)
  const uint64_t* hat = nullptr;
  const uint64_t* big_p = nullptr;
  const uint64_t* half_p = nullptr;
  int p_limbs = 0;
};
// Ambiguity list for icrt(): counter + coefficient ids whose fp64 quotient
// lies within 1/4 of a half-integer, i.e. |v| >= P/4 — impossible inside
// he_mul (slack >= 4 bits is asserted at level setup), possible for
// arbitrary residues passed to the stage API. Those coefficients are
// recomputed exactly by a fix-up kernel.
struct IcrtFlags {
  unsigned* count = nullptr;  // device counter, zeroed by icrt()
  unsigned* ids = nullptr;    // capacity entries: b * n + i
  unsigned capacity = 0;
};
cudaError_t icrt_setup_attributes();
// rns: batch x np x n canonical residues; out: batch x n x ceil(T/64) limbs.
// flags = nullptr: the caller guarantees |v| < P/4 (he_mul).
// rns_hi (split region 1, no flags): out = c0 + 2^h c1 mod 2^T for c0 = rns,
// c1 = rns_hi, with the table of a split region (level_tables.hpp).
template <class F>
cudaError_t icrt(const typename F::W* rns, size_t batch, int log_n,
                 const typename F::Prime* primes, int np, const IcrtTable& t, uint64_t* out,
                 cudaStream_t st, const IcrtFlags* flags = nullptr,
                 const typename F::W* rns_hi = nullptr);

// Fused key-switch finisher (heaan.cpp:398-409 after the evk product): for
// each coefficient one GEMM over the region-2 residues of ks (t_j halves + k)
// and the region-1 residues of d evaluates
//   V = X2 + 2^(logQ-1) + 2^logQ (X1 + 2^(logp-1)),
//   X2 = ks-part mod 2^(logq+logQ), X1 = d mod 2^logq,
// from bit `base` up, and writes out = bits [logQ+logp, logQ+logq) of V
// = R_logp(d + R_logQ(ks)) — ModDown, the add and the rescale at once.
// Region-2 rows are truncated below bit base = logQ - 125; the dropped part
// is < 2^(base+68), so a coefficient is exact unless the 64 bits below the
// output are all ones (probability 2^-64); such coefficients are flagged and
// recomputed by an exact big-integer fix-up kernel (no approximation ever
// reaches the output).
struct Finisher {
  const uint32_t* btab = nullptr;  // (k2 + k1) x cols_pad, 25-bit chunks
  int cols = 0, cols_pad = 0, k2 = 0, k1 = 0, base = 0;
  int half_q_bit = 0, half_p_bit = 0, out_bit = 0, out_bits = 0;
  int log_q = 0, log_Q = 0, log_p = 0;
  // split region 1 (level_tables.hpp): d = c0 + 2^split_h c1, c1 stored
  // hi_off residues after c0; hi_off = 0: unsplit
  int split_h = 0;
  size_t hi_off = 0;
  int t_inputs = 0;  // residues are t_j already (tensor-core path, bigint_tc.cu)
  int tS = 0;        // residue rows column-major (BigTcOut::tS); flag ids per coefficient
};
cudaError_t finisher_setup_attributes();
// ks: 2B x np2 x n (B ax-batches then B bx-batches), d_ax / d_bx: B x np1 x n
// (iNTT'd d1 / d0); out: B x n x ceil((logq-logp)/64) each.
// force_exact != 0 routes every coefficient through the exact fix-up (test).
template <class F>
cudaError_t finish_keyswitch(const typename F::W* ks, const typename F::W* d_ax,
                             const typename F::W* d_bx, size_t B, int log_n,
                             const typename F::Prime* p2, int np2, const typename F::Prime* p1,
                             int np1, const Finisher& f,
                             const IcrtTable& t2, const IcrtTable& t1, uint64_t* out_ax,
                             uint64_t* out_bx, const IcrtFlags& flags, int force_exact,
                             cudaStream_t st);

// ---- iCRT / key-switch finisher on the int8 tensor cores (bigint_tc.cu) -----
// One RNS operand feeding the GEMM's A rows (t_j residues, prime-major rows
// of n): entry e (< entries) reads rows row0 + (e % B) erows + (e >= B ?
// half_rows : 0) + j (j < np) of raw tensor map `map` (bigint_tc's rmaps).
struct BigTcSeg {
  int map = 0;
  int row0 = 0, erows = 0, half_rows = 0;
  const DevPrime32* primes = nullptr;  // pad[0] = floor(2^55 / p) (the k quotient)
  int np = 0;
  int slot0 = 0;  // set from the table
};
// Constant GEMM operand (level_tables.cpp build_bigint): B[m][K] u8, column
// m <-> 2^(8 (m + m0)) of the window; segment s's row j occupies K bytes
// 4 (slot0[s] + j) .. +3, the k quotients bytes 4 k_slot + 2 s, +1. Stored
// chunk-major and pre-swizzled: btab = [k_bytes / 64][n_cols][64].
struct BigTcTable {
  const uint8_t* btab = nullptr;
  int n_cols = 0;   // multiple of 32, <= 480 (16-column TMEM reads past the end)
  int k_bytes = 0;  // multiple of 64
  int k_slot = 0;
  int nseg = 0;
  int slot0[3] = {0, 0, 0}, np[3] = {0, 0, 0};
};
// Output window: limbs of bits [out_bit, out_bit + out_bits) of the window
// value (rounding constants included by the table) to out0 (entries < B) / out1 (>= B),
// n x out_limbs per entry. check_amb: coefficients whose 64 bits below
// out_bit are all ones (truncated window, p = 2^-64) and, with force_exact,
// every coefficient, are listed in flags and left to the exact fix-up.
struct BigTcOut {
  uint64_t* out0 = nullptr;
  uint64_t* out1 = nullptr;
  int out_limbs = 0, out_bit = 0, out_bits = 0;
  int check_amb = 0, force_exact = 0;
  // tS > 0: the t rows are in NTT pass A's column-major layout (position
  // x 2^tS + y holds coefficient y n / 2^tS + x); outputs and flag ids are
  // per coefficient either way
  int tS = 0;
  IcrtFlags flags;
};
cudaError_t bigint_tc_setup_attributes();
size_t bigint_tc_smem(int n_cols);
bool bigint_tc_supported(int n_cols);
// rmaps[2]: host pointers to CUtensorMaps of u32 residue arrays [rows][n]
// (box 128 x 16, no swizzle; make_raw_tmap).
cudaError_t bigint_tc(const BigTcTable& t, const BigTcSeg* segs, int entries, int B, int log_n,
                      const BigTcOut& o, const void* const* rmaps, cudaStream_t st);
// Exact fix-up of flagged finisher coefficients (icrt.cu finish_fixup_kernel).
template <class F>
cudaError_t finish_fixup(const typename F::W* ks, const typename F::W* d_ax,
                         const typename F::W* d_bx, size_t B, int log_n,
                         const typename F::Prime* p2, int np2, const typename F::Prime* p1,
                         int np1, const Finisher& f, const IcrtTable& t2, const IcrtTable& t1,
                         uint64_t* out_ax, uint64_t* out_bx, const IcrtFlags& flags,
                         cudaStream_t st);

// ---- element-wise RNS and polynomial kernels (poly.cu) ---------------------
// out = a * b mod p_j over batch x np x n.
cudaError_t pointwise(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t batch, int np,
                      int log_n, const DevPrime* primes, cudaStream_t st);
// Region-1 tensor product in the evaluation domain (heaan.cpp:372-394 with
// the cross term as A1 B2 + A2 B1, bit-identical to the (a+b)(a'+b') form,
// test_heaan.cpp:184-199): d0 = B1 B2, d2 = A1 A2, d1 = A1 B2 + A2 B1.
template <class F>
cudaError_t tensor_product(const typename F::W* a1, const typename F::W* b1,
                           const typename F::W* a2, const typename F::W* b2, typename F::W* d0,
                           typename F::W* d1, typename F::W* d2, size_t batch, int np,
                           int log_n, const typename F::Prime* primes, cudaStream_t st);
// Split region 1 (F32::tensor_split) for the unfused path: r1 = 8 slots of
// batch x np x n; the six half products land in slots 0..5.
cudaError_t tensor_split_product(uint32_t* r1, size_t batch, int np, int log_n,
                                 const DevPrime32* primes, cudaStream_t st);
// Region-2 evk inner product: ka = f * ea, kb = f * eb (evk forms shared by
// the batch).
template <class F>
cudaError_t evk_product(const typename F::W* f, const typename F::W* ea, const typename F::W* eb,
                        typename F::W* ka, typename F::W* kb, size_t batch, int np, int log_n,
                        const typename F::Prime* primes, cudaStream_t st);
// out = R_logp( d + R_logQ(ks) mod 2^log_q ): ModDown shift, add and rescale
// (poly.cpp:98-115, heaan.cpp:401-409). ks: n x ceil((log_q+log_Q)/64),
// d: n x ceil(log_q/64), out: n x ceil((log_q-log_p)/64); batch of each.
cudaError_t keyswitch_epilogue(const uint64_t* ks, const uint64_t* d, uint64_t* out, size_t batch,
                               int log_n, int log_q, int log_Q, int log_p, cudaStream_t st);
// rows x cols words -> cols x rows (BigPoly coefficient-major <-> limb-major)
cudaError_t word_transpose(const uint64_t* in, uint64_t* out, int rows, int cols, cudaStream_t st);
// Scheme::mul_by_ternary (heaan.cpp:234-256) on limb-major polys (L x n):
// nz[j] = 2 i_j + (s_j < 0) lists the nonzero ternary coefficients.
cudaError_t mul_by_ternary(const uint64_t* aT, const int* nz, int nnz, uint64_t* rT, int log_n,
                           int log_q, cudaStream_t st);
// poly_mod_down (poly.cpp:117-127) on a poly batch: n x ceil(log_q/64) ->
// n x ceil(new_log_q/64), top limb masked.
cudaError_t mod_down(const uint64_t* a, uint64_t* out, size_t batch, int log_n, int log_q,
                     int new_log_q, cudaStream_t st);
// Scheme::rescale on one poly batch (poly_shift_right, poly.cpp:98-115).
cudaError_t shift_right(const uint64_t* a, uint64_t* out, size_t batch, int log_n, int log_q,
                        int bits, cudaStream_t st);

}  // namespace hemul_gpu
