// Host-callable launchers of the sm_100a kernels (one .cu file per stage).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "device_tables.cuh"

namespace hemul_gpu {

// Opt-in dynamic shared memory cap we request (227 KB per CTA minus room for
// static shared arrays).
constexpr int kMaxDynSmem = 224 * 1024;

// ---- NTT (ntt.cu) ----------------------------------------------------------
cudaError_t ntt_setup_attributes();
// rows = batch * np prime-major rows; row r uses prime r % np.
cudaError_t ntt_forward(uint64_t* data, size_t rows, int np, int log_n, const Twiddle* tw,
                        const DevPrime* primes, cudaStream_t st, int* launches);
cudaError_t ntt_inverse(uint64_t* data, size_t rows, int np, int log_n, const Twiddle* itw,
                        const DevPrime* primes, cudaStream_t st, int* launches);
// The same transforms one memory pass at a time (for per-kernel timing):
// forward pass 0 = levels [0, s1) on columns, pass 1 = levels [s1, logN) on
// blocks; inverse pass 0 = levels [s1, logN), pass 1 = levels [0, s1) + n^-1.
int ntt_num_passes(int log_n);
cudaError_t ntt_forward_pass(int pass, uint64_t* data, size_t rows, int np, int log_n,
                             const Twiddle* tw, const DevPrime* primes, cudaStream_t st);
cudaError_t ntt_inverse_pass(int pass, uint64_t* data, size_t rows, int np, int log_n,
                             const Twiddle* itw, const DevPrime* primes, cudaStream_t st);

// Fused middle pass (two-pass sizes, logN 12..17): forward levels
// [s1, logN) of every operand + the evaluation-domain product + inverse
// levels [s1, logN) of the products, one read and one write per block.
// Inputs come out of forward pass 0, outputs go into inverse pass 1.
bool ntt_has_mid(int log_n);
// Region 1: A1 B1 A2 B2 -> d2 (over A1), d0 (over B1), d1 = A1B2 + A2B1 (over A2).
cudaError_t ntt_mid_tensor(uint64_t* A1, uint64_t* B1, uint64_t* A2, uint64_t* B2, size_t batch,
                           int np, int log_n, const Twiddle* tw, const Twiddle* itw,
                           const DevPrime* primes, cudaStream_t st);
// Region 2: F -> F evk_a (KA), F evk_b (KB); KA may alias F.
cudaError_t ntt_mid_evk(uint64_t* F, const uint64_t* ea, const uint64_t* eb, uint64_t* KA,
                        uint64_t* KB, size_t batch, int np, int log_n, const Twiddle* tw,
                        const Twiddle* itw, const DevPrime* primes, cudaStream_t st);

// ---- integer-pipe peak probe (probe.cu) ------------------------------------
// Measured IMAD.WIDE.U32 throughput of this device in ops/s (a dependent-free
// stream of mad.wide.u32, 148 x 8 CTAs), and the SM clock it ran at (kHz).
cudaError_t imad_peak(double* ops_per_s, cudaStream_t st);

// ---- CRT (crt.cu) ----------------------------------------------------------
// Weight table for one (prime set, input width): wtab[m * ld + 2 j + h]
// = 30-bit half h of 2^(25 m) mod p_j, m < chunks = ceil(in_bits / 25)
// (the input is cut into 25-bit chunks: the iGEMM operand widths).
struct CrtWeights {
  const uint32_t* wtab = nullptr;
  int chunks = 0;
  int ld = 0;  // crt_cols_pad(2 np)
};
constexpr int kCrtPrimesPerTile = 16;
cudaError_t crt_setup_attributes();
// poly: batch x n x limbs; out: batch x np x n.
cudaError_t crt_forward(const uint64_t* poly, int limbs, size_t batch, int log_n,
                        const CrtWeights& w, const DevPrime* primes, int np, uint64_t* out,
                        cudaStream_t st);
// Up to 4 independent inputs of `batch` polys each in one launch; input t
// lands at out + t * batch * np * n.
cudaError_t crt_forward_multi(const uint64_t* const* polys, int count, int limbs, size_t batch,
                              int log_n, const CrtWeights& w, const DevPrime* primes, int np,
                              uint64_t* out, cudaStream_t st);

// ---- iCRT (icrt.cu) --------------------------------------------------------
// B table for the exact reconstruction mod 2^T: (2 np + 1) rows x m_pad
// columns of 25-bit chunks (rows 2j: H_j mod 2^T, 2j+1: H_j 2^30 mod 2^T,
// 2np: (-P) mod 2^T), m_out = ceil(T / 25) real columns.
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
cudaError_t icrt(const uint64_t* rns, size_t batch, int log_n, const DevPrime* primes, int np,
                 const IcrtTable& t, uint64_t* out, cudaStream_t st,
                 const IcrtFlags* flags = nullptr);

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
};
cudaError_t finisher_setup_attributes();
// ks: 2B x np2 x n (B ax-batches then B bx-batches), d_ax / d_bx: B x np1 x n
// (iNTT'd d1 / d0); out: B x n x ceil((logq-logp)/64) each.
// force_exact != 0 routes every coefficient through the exact fix-up (test).
cudaError_t finish_keyswitch(const uint64_t* ks, const uint64_t* d_ax, const uint64_t* d_bx,
                             size_t B, int log_n, const DevPrime* p2, int np2,
                             const DevPrime* p1, int np1, const Finisher& f,
                             const IcrtTable& t2, const IcrtTable& t1, uint64_t* out_ax,
                             uint64_t* out_bx, const IcrtFlags& flags, int force_exact,
                             cudaStream_t st);

// ---- element-wise RNS and polynomial kernels (poly.cu) ---------------------
// out = a * b mod p_j over batch x np x n.
cudaError_t pointwise(const uint64_t* a, const uint64_t* b, uint64_t* out, size_t batch, int np,
                      int log_n, const DevPrime* primes, cudaStream_t st);
// Region-1 tensor product in the evaluation domain (heaan.cpp:372-394 with
// the cross term as A1 B2 + A2 B1, bit-identical to the (a+b)(a'+b') form,
// test_heaan.cpp:184-199): d0 = B1 B2, d2 = A1 A2, d1 = A1 B2 + A2 B1.
cudaError_t tensor_product(const uint64_t* a1, const uint64_t* b1, const uint64_t* a2,
                           const uint64_t* b2, uint64_t* d0, uint64_t* d1, uint64_t* d2,
                           size_t batch, int np, int log_n, const DevPrime* primes,
                           cudaStream_t st);
// Region-2 evk inner product: ka = f * ea, kb = f * eb (evk forms shared by
// the batch).
cudaError_t evk_product(const uint64_t* f, const uint64_t* ea, const uint64_t* eb, uint64_t* ka,
                        uint64_t* kb, size_t batch, int np, int log_n, const DevPrime* primes,
                        cudaStream_t st);
// out = R_logp( d + R_logQ(ks) mod 2^log_q ): ModDown shift, add and rescale
// (poly.cpp:98-115, heaan.cpp:401-409). ks: n x ceil((log_q+log_Q)/64),
// d: n x ceil(log_q/64), out: n x ceil((log_q-log_p)/64); batch of each.
cudaError_t keyswitch_epilogue(const uint64_t* ks, const uint64_t* d, uint64_t* out, size_t batch,
                               int log_n, int log_q, int log_Q, int log_p, cudaStream_t st);
// Scheme::rescale on one poly batch (poly_shift_right, poly.cpp:98-115).
cudaError_t shift_right(const uint64_t* a, uint64_t* out, size_t batch, int log_n, int log_q,
                        int bits, cudaStream_t st);

}  // namespace hemul_gpu
