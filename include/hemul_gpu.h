/* hemul_gpu.h — C-ABI of the B200 HE Mul path (libhemul_gpu.so).
 *
 * The reference (/root/reference/proj, "hemul") has no FFI: its boundary is the
 * C++ API in namespace hemul. Each entry point below replaces one reference
 * interface, cited as file:line (paths relative to proj/core/):
 *
 *   hemul_gpu_create        Scheme::Scheme(const Params&)        include/hemul/heaan.hpp:74
 *                           + make_params                        src/params.cpp:64-74
 *   hemul_gpu_set_level     Scheme::warm_level(log_q, nullptr)   include/hemul/heaan.hpp:100
 *                           (Scheme::level, tables only)         src/heaan.cpp:119-150
 *   hemul_gpu_set_evk       Scheme::warm_level(log_q, &evk)      src/heaan.cpp:152-167
 *   hemul_gpu_he_mul        Scheme::he_mul(c1, c2, evk)          include/hemul/heaan.hpp:91-92,
 *                                                                src/heaan.cpp:339-410
 *   hemul_gpu_rescale       Scheme::rescale(c)                   src/heaan.cpp:328-337
 *   hemul_gpu_stage_ms      Scheme::timers (StageTimers)         include/hemul/counters.hpp:13,44-57
 *   hemul_gpu_ntt / _crt /  ntt_forward / ntt_inverse            include/hemul/ntt.hpp:34-39
 *   _icrt / _pointwise      crt_forward / icrt_reordered /       include/hemul/rns.hpp:62-85
 *                           rns_pointwise_mul
 *   hemul_gpu_level_info    PrimeSet / region{1,2}_prime_count   include/hemul/params.hpp:39-67
 *
 * Conventions
 *  - Polynomials use the reference BigPoly layout (poly.hpp:15-26): n x limbs
 *    u64, data[i*limbs + k], little-endian 64-bit limbs, limbs =
 *    ceil(log_q/64), top limb masked. Batches are `batch` such polynomials
 *    back to back.
 *  - RNS matrices are prime-major, data[j*n + i] (rns.hpp:17-20 Layout::
 *    prime_major); batches back to back.
 *  - Every pointer may be host memory (pageable or pinned) or device memory
 *    of the context's GPU; the library detects which with
 *    cudaPointerGetAttributes and copies as needed on the context stream.
 *  - No exceptions cross this boundary. Errors are status codes mirroring the
 *    reference's exception kinds; hemul_gpu_last_error returns the message
 *    (identical to the reference's what() string where one exists).
 *  - A context is not thread safe (Scheme::he_mul is non-const, heaan.hpp:
 *    91-92): use one per host thread or serialize.
 *  - There is no CPU fallback: without a usable CUDA device every call that
 *    computes returns HEMUL_E_CUDA.
 */
#ifndef HEMUL_GPU_H
#define HEMUL_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hemul_gpu_ctx hemul_gpu_ctx;

typedef enum {
  HEMUL_OK = 0,
  HEMUL_E_ARG = 1,               /* std::invalid_argument (bad size, layout, radix...) */
  HEMUL_E_MODULUS_MISMATCH = 2,  /* "ciphertext modulus mismatch"   heaan.cpp:341-342 */
  HEMUL_E_DEPTH = 3,             /* "multiplicative depth exhausted" heaan.cpp:344-345
                                    "modulus exhausted; cannot rescale" heaan.cpp:329-330 */
  HEMUL_E_CUDA = 4,              /* CUDA runtime / launch failure, or no device */
  HEMUL_E_OOM = 5,               /* device allocation failed */
  HEMUL_E_NO_EVK = 6,            /* he_mul before set_evk at this level */
  HEMUL_E_IO = 7                 /* IoError: unreadable / corrupt / truncated file (io.cpp) */
} hemul_status;

/* Stage buckets, same order as hemul::Stage (counters.hpp:13). */
enum { HEMUL_STAGE_CRT = 0, HEMUL_STAGE_NTT, HEMUL_STAGE_INTT, HEMUL_STAGE_ICRT,
       HEMUL_STAGE_EXTRA, HEMUL_STAGE_COUNT };

/* Kernel classes for per-launch device timing (hemul_gpu_kernel_stats). */
enum { HEMUL_KCLASS_CRT = 0, HEMUL_KCLASS_NTT_A, HEMUL_KCLASS_NTT_B, HEMUL_KCLASS_INTT_B,
       HEMUL_KCLASS_INTT_A, HEMUL_KCLASS_TENSOR, HEMUL_KCLASS_EVK, HEMUL_KCLASS_ICRT,
       HEMUL_KCLASS_FINISH, HEMUL_KCLASS_MID_R1, HEMUL_KCLASS_MID_R2, HEMUL_KCLASS_EPILOGUE,
       HEMUL_KCLASS_H2D, HEMUL_KCLASS_D2H, HEMUL_KCLASS_COUNT };

/* make_params(log_p, depth, w64, log_n_override) (params.cpp:64-74) and a
 * context on CUDA device `device`. log_n_override = 0 uses the security table
 * (params.cpp:56-62). */
hemul_status hemul_gpu_create(int device, int log_p, int depth, int log_n_override,
                              hemul_gpu_ctx **out);
void hemul_gpu_destroy(hemul_gpu_ctx *ctx);
const char *hemul_gpu_last_error(const hemul_gpu_ctx *ctx);
/* {log_n, n, log_p, depth, log_q_max} */
hemul_status hemul_gpu_params(const hemul_gpu_ctx *ctx, int out[5]);

/* Launch everything on `stream` (a cudaStream_t of the context's device;
 * NULL = the context's own stream). Lets a caller (e.g. PyTorch) order the
 * library's kernels with its own work and time them with its own events. */
hemul_status hemul_gpu_set_stream(hemul_gpu_ctx *ctx, void *stream);

/* Build (or fetch from the 2-entry LRU, heaan.cpp:119-150) the tables of
 * modulus log_q. */
hemul_status hemul_gpu_set_level(hemul_gpu_ctx *ctx, int log_q);

/* Cache the evaluation key's region-2 NTT forms at level log_q
 * (heaan.cpp:152-167). evk polys: n x ceil(2 log_q_max / 64) limbs. evk_id
 * identifies the key (the reference compares the EvalKey address,
 * heaan.cpp:152; here the caller passes any stable id, 0 = always rebuild). */
hemul_status hemul_gpu_set_evk(hemul_gpu_ctx *ctx, int log_q, const uint64_t *evk_ax,
                               const uint64_t *evk_bx, uint64_t evk_id);

/* batch independent HE Muls: out_b = rescale(relinearize(c1_b * c2_b))
 * (heaan.cpp:339-410). Inputs n x ceil(log_q/64) limbs per poly; outputs
 * n x ceil((log_q - log_p)/64). Checks run in the reference's order:
 * c1_log_q != c2_log_q -> HEMUL_E_MODULUS_MISMATCH; log_q - log_p < log_p ->
 * HEMUL_E_DEPTH. The evk must have been set at this level (or is set from
 * evk_ax/evk_bx when those are non-null). */
hemul_status hemul_gpu_he_mul(hemul_gpu_ctx *ctx, int c1_log_q, int c2_log_q, size_t batch,
                              const uint64_t *c1_ax, const uint64_t *c1_bx,
                              const uint64_t *c2_ax, const uint64_t *c2_bx,
                              const uint64_t *evk_ax, const uint64_t *evk_bx, uint64_t evk_id,
                              uint64_t *out_ax, uint64_t *out_bx);

/* Which kernels he_mul runs at level log_q (the basis and engine choice are
 * per level: table shapes change with log_q). Fills info[HEMUL_INFO_*]. */
enum { HEMUL_INFO_WORD = 0,     /* 32 (30-bit basis) or 64 (reference primes) */
       HEMUL_INFO_NP1,          /* region-1 primes (per half product when split) */
       HEMUL_INFO_NP2,          /* region-2 primes */
       HEMUL_INFO_SPLIT_H,      /* region-1 operand split bit h (0: unsplit) */
       HEMUL_INFO_CRT1_TC,      /* region-1 CRT on the int8 tensor cores */
       HEMUL_INFO_CRT2_TC,      /* ModUp CRT on the tensor cores */
       HEMUL_INFO_BIG_TC,       /* iCRT + finisher on the tensor cores (t_j form) */
       HEMUL_INFO_FUSED_MID,    /* fused middle NTT pass with the products */
       HEMUL_INFO_BLK_MONT,     /* Montgomery-reduced warp-per-block middle pass */
       HEMUL_INFO_T_PASS_A,     /* > 0: CRT outputs and t rows are column-major with
                                   this pass-A level count S (HEMUL_OPT_TRANSPOSED):
                                   position x 2^S + y holds coefficient y n / 2^S + x
                                   (he_mul_trace checkpoints crt1, prod1, crt2, prod2) */
       HEMUL_INFO_COUNT };
hemul_status hemul_gpu_engine_info(hemul_gpu_ctx *ctx, int log_q, int info[HEMUL_INFO_COUNT]);

/* Test hook: run he_mul on `batch` pairs up to a stage checkpoint and copy
 * that stage's device buffer to dst (host or device, cap bytes); *written =
 * bytes copied. Lets the residue-level tests check the hot-path kernels of
 * the 30-bit basis stage by stage against the restated oracle (the stage
 * entry points below use the reference's w64 primes). Layouts (W = 4-byte
 * residues in the 30-bit basis, 8 in w64; rows prime-major, n residues):
 *   CRT1  region-1 operands after the CRT: 8 slots (w64: 4) of batch x np1
 *         rows; slots x1 X1 y1 Y1 x2 X2 y2 Y2 = low / high halves (split at
 *         h) of ax1 bx1 ax2 bx2 (w64: ax1 bx1 ax2 bx2); residues in [0, 2p)
 *   PROD1 the products after the inverse NTT: 6 slots (w64: 3) of batch x
 *         np1 rows, x1x2, x1X2+X1x2, y1y2, y1Y2+Y1y2, x1y2+x2y1,
 *         x1Y2+X1y2+x2Y1+X2y1 (w64: d2, d0, d1); residues x_j, or t_j =
 *         x_j (P/p_j)^-1 when HEMUL_INFO_BIG_TC
 *   D2    d2 = ax1 ax2 mod 2^log_q, batch BigPolys (n x ceil(log_q/64))
 *   CRT2  d2 in the region-2 primes: batch x np2 rows, [0, 2p)
 *   PROD2 the evk products after the inverse NTT: 2 x batch x np2 rows
 *         (d2 evk.ax, then d2 evk.bx), x_j or t_j as PROD1 */
enum { HEMUL_TRACE_CRT1 = 1, HEMUL_TRACE_PROD1, HEMUL_TRACE_D2, HEMUL_TRACE_CRT2,
       HEMUL_TRACE_PROD2 };
hemul_status hemul_gpu_he_mul_trace(hemul_gpu_ctx *ctx, int log_q, size_t batch,
                                    const uint64_t *c1_ax, const uint64_t *c1_bx,
                                    const uint64_t *c2_ax, const uint64_t *c2_bx,
                                    const uint64_t *evk_ax, const uint64_t *evk_bx,
                                    uint64_t evk_id, int checkpoint, void *dst, size_t cap,
                                    size_t *written);

/* ---- device-resident ciphertexts (HE Mul chains without host copies) -----
 * The reference's Ciphertext is a host value (heaan.hpp:38-42); a chain such
 * as the multiplication ladder (test_heaan.cpp:143-167) copies every operand
 * and result across PCIe when driven through hemul_gpu_he_mul with host
 * buffers. A handle keeps a batch of ciphertexts {ax, bx, log_q} in device
 * memory (stream-ordered pool); the operations below queue kernels on the
 * context stream and return without waiting; only create (from host memory)
 * and download synchronise. Results are new handles; the caller destroys
 * every handle it receives (hemul_gpu_ct_destroy, ordered on ctx's stream;
 * ctx = NULL frees synchronously). */
typedef struct hemul_gpu_ct hemul_gpu_ct;
/* batch ciphertexts at modulus log_q from BigPoly buffers (host or device;
 * NULL = zero polynomials). flags = 0: returns after the copy (the sources
 * may be reused at once). HEMUL_CT_ASYNC: the copy is queued on the
 * context's copy stream and overlaps kernels already queued; later work on
 * the handle waits for it; pinned sources must stay unchanged until the next
 * synchronising call (download / hemul_gpu_synchronize). */
enum { HEMUL_CT_ASYNC = 1 };
hemul_status hemul_gpu_ct_create(hemul_gpu_ctx *ctx, int log_q, size_t batch,
                                 const uint64_t *ax, const uint64_t *bx, int flags,
                                 hemul_gpu_ct **out);
void hemul_gpu_ct_destroy(hemul_gpu_ctx *ctx, hemul_gpu_ct *ct);
hemul_status hemul_gpu_ct_info(const hemul_gpu_ct *ct, int *log_q, size_t *batch);
/* device addresses of the ax / bx batches (n x ceil(log_q/64) words each per
 * ciphertext), e.g. to wrap them in framework tensors */
hemul_status hemul_gpu_ct_device_ptrs(const hemul_gpu_ct *ct, uint64_t **ax, uint64_t **bx);
hemul_status hemul_gpu_ct_download(hemul_gpu_ctx *ctx, const hemul_gpu_ct *ct, uint64_t *ax,
                                   uint64_t *bx);
/* HEA1 ciphertext files (io.cpp:101-141) straight to / from HBM through a
 * pinned double buffer (the file read / write of chunk k overlaps the PCIe
 * copy of chunk k+1): load_ciphertext + upload, download + save_ciphertext.
 * 64-bit words at the context's ring degree; batch-1 handles. */
hemul_status hemul_gpu_ct_load(hemul_gpu_ctx *ctx, const char *path, hemul_gpu_ct **out,
                               int *n_slots);
hemul_status hemul_gpu_ct_save(hemul_gpu_ctx *ctx, const hemul_gpu_ct *ct, int n_slots,
                               const char *path);
/* Scheme::he_mul (heaan.cpp:339-410) on two handles of equal batch; same
 * checks and errors as hemul_gpu_he_mul; *out at log_q - log_p. */
hemul_status hemul_gpu_ct_he_mul(hemul_gpu_ctx *ctx, const hemul_gpu_ct *c1,
                                 const hemul_gpu_ct *c2, const uint64_t *evk_ax,
                                 const uint64_t *evk_bx, uint64_t evk_id, hemul_gpu_ct **out);
/* Scheme::rescale (heaan.cpp:328-337) */
hemul_status hemul_gpu_ct_rescale(hemul_gpu_ctx *ctx, const hemul_gpu_ct *ct, hemul_gpu_ct **out);
/* poly_mod_down (poly.cpp:117-127) of both polynomials to new_log_q <= log_q:
 * the ladder's modulus alignment (test_heaan.cpp:154-160) */
hemul_status hemul_gpu_ct_mod_down(hemul_gpu_ctx *ctx, const hemul_gpu_ct *ct, int new_log_q,
                                   hemul_gpu_ct **out);

/* Scheme::mul_by_ternary (heaan.cpp:234-256): out_b = a_b * t mod (X^n + 1,
 * 2^log_q) for batch BigPolys a_b (n x ceil(log_q/64)) and one ternary
 * polynomial t (n int32 in {-1, 0, 1}, typically sparse: the secret key or
 * the encryption randomness). The key generation, encryption and decryption
 * products of the drop-in Scheme run here; the RNG stays on the host so the
 * keys follow the reference's transcript (rng.hpp). */
hemul_status hemul_gpu_mul_by_ternary(hemul_gpu_ctx *ctx, int log_q, size_t batch,
                                      const uint64_t *a, const int32_t *t, uint64_t *out);

/* Scheme::rescale (heaan.cpp:328-337) on a batch: n x ceil(log_q/64) ->
 * n x ceil((log_q - log_p)/64). */
hemul_status hemul_gpu_rescale(hemul_gpu_ctx *ctx, int log_q, size_t batch, const uint64_t *ax,
                               const uint64_t *bx, uint64_t *out_ax, uint64_t *out_bx);

/* Options. HEMUL_OPT_FORCE_EXACT = 1 routes every output coefficient of
 * he_mul through the exact big-integer fix-up kernel that normally only
 * handles the (probability 2^-64) coefficients whose truncated ModDown window
 * is ambiguous — a test knob for that path; results are identical.
 * HEMUL_OPT_BASIS selects the RNS prime basis he_mul computes in: 32 (the
 * default) = primes p = 1 mod 2n below 2^30 with 32-bit residues, 64 = the
 * reference's own w64 primes (params.cpp:89-115). The product is exact in
 * either basis, so the ciphertexts are bit-identical; the 30-bit basis falls
 * back to 64 when a ring degree has too few such primes. Changing it
 * invalidates cached evk forms (pass the evk to the next he_mul).
 * HEMUL_OPT_TENSOR_CORES (default 1): in the 30-bit basis the big-integer
 * base conversions run as exact u8 x u8 -> s32 GEMMs on the tcgen05 tensor
 * cores; 0 selects the IMAD.WIDE integer-pipe kernels. Results are
 * bit-identical either way. */
enum { HEMUL_OPT_FORCE_EXACT = 1, HEMUL_OPT_BASIS = 2, HEMUL_OPT_TENSOR_CORES = 3,
       HEMUL_OPT_LEVEL_CACHE = 4, HEMUL_OPT_TRANSPOSED = 5 };
/* HEMUL_OPT_TRANSPOSED: in the tensor-core engine at log N >= 15 the RNS rows
 * around NTT pass A use the column-major layout (CRT writes it, the forward
 * column pass reads it without a staging barrier, the inverse column pass
 * writes it without a store phase, the iCRT / finisher read it). Results are
 * identical either way. Default 1. */
/* HEMUL_OPT_LEVEL_CACHE: capacity of the level LRU (default 2, the
 * reference's Scheme::level, heaan.cpp:119-150). A device-resident chain
 * walks one level per HE Mul; with a larger cache (about 1 GB per level at
 * N=2^17) a repeated chain keeps every level's tables and evk forms. */
hemul_status hemul_gpu_set_option(hemul_gpu_ctx *ctx, int option, int value);

/* Device timing. When enabled every launch is bracketed by CUDA events on the
 * context stream (read back lazily, so no extra host sync per call).
 * stage_ms: per-stage milliseconds of the last he_mul call, buckets as
 * counters.hpp:13 (pointwise booked under iCRT like rns.cpp:364).
 * kernel_stats: cumulative milliseconds and launch counts per kernel class
 * since the last reset_stats. */
hemul_status hemul_gpu_enable_stage_timing(hemul_gpu_ctx *ctx, int on);
hemul_status hemul_gpu_stage_ms(hemul_gpu_ctx *ctx, double ms[HEMUL_STAGE_COUNT]);
hemul_status hemul_gpu_kernel_stats(hemul_gpu_ctx *ctx, double ms[HEMUL_KCLASS_COUNT],
                                    uint64_t launches[HEMUL_KCLASS_COUNT]);
hemul_status hemul_gpu_reset_stats(hemul_gpu_ctx *ctx);

/* Integer-pipe roofline denominator: measured IMAD.WIDE.U32 ops/s of the
 * context's device (a short probe kernel). */
hemul_status hemul_gpu_imad_peak(hemul_gpu_ctx *ctx, double *ops_per_s);
/* Tensor-core roofline denominator: measured dense int8 ops/s (2 per u8 x u8
 * MAC) of tcgen05.mma kind::i8 on the context's device, the engine of the
 * 30-bit basis' CRT / iCRT / finisher GEMMs (HEMUL_OPT_TENSOR_CORES). */
hemul_status hemul_gpu_tc_peak(hemul_gpu_ctx *ctx, double *ops_per_s);

/* Prime set of level log_q: region 1 (products mod q) or 2 (key switching)
 * by the reference's w64 rule (params.cpp:76-115, heaan.cpp:132-143) —
 * host arithmetic only, no tables are built or uploaded; region -1 / -2: the
 * basis he_mul runs in (HEMUL_OPT_BASIS; builds that level's tables). Writes
 * np and up to cap primes. */
hemul_status hemul_gpu_level_info(hemul_gpu_ctx *ctx, int log_q, int region, int *np,
                                  uint64_t *primes, int cap);

/* ---- stage entry points (the reference's lower-level API) ---------------- */

/* ntt_forward / ntt_inverse (ntt.cpp:153-197) in place over `rows` prime-major
 * rows of n residues; row r is transformed mod prime (r % np) of the region. */
hemul_status hemul_gpu_ntt(hemul_gpu_ctx *ctx, int log_q, int region, uint64_t *data, size_t rows,
                           int inverse);
/* ntt_forward / ntt_inverse (ntt.cpp:59-137, 153-197) in the B200 30-bit
 * basis of a level (hemul_gpu_level_info region -1 / -2 lists its primes):
 * rows of n u32 residues, row r mod prime r % np over the basis' first np
 * primes (np = 0: all of them), the column / block kernels of the he_mul
 * path (pass A ntt_col.cu + pass B), outputs in the lazy ranges of the
 * 30-bit field ([0, 4p) forward, [0, p) inverse). For the C2 NTT sweep and
 * residue-level tests. */
hemul_status hemul_gpu_ntt32(hemul_gpu_ctx *ctx, int log_q, int region, int np, uint32_t *data,
                             size_t rows, int inverse);
/* make_ntt_tables (params.cpp:151-180) of the level's 30-bit basis, built on
 * the device: prime j's forward and inverse twiddles as n (w, wq) u32 pairs
 * each, tw[rev(i)] = psi_j^i, itw[rev(i)] = psi_j^-i, wq = floor(w 2^32 / p_j)
 * (either output may be NULL). Introspection for tests. */
hemul_status hemul_gpu_level_twiddles32(hemul_gpu_ctx *ctx, int log_q, int region, int j,
                                        uint32_t *tw, uint32_t *itw);
/* crt_forward (rns.cpp:331-358): batch polys of n x ceil(in_bits/64) limbs ->
 * batch x np x n residues. */
hemul_status hemul_gpu_crt(hemul_gpu_ctx *ctx, int log_q, int region, int in_bits, size_t batch,
                           const uint64_t *poly, uint64_t *rns);
/* rns_pointwise_mul (rns.cpp:360-371) on batch x np x n. */
hemul_status hemul_gpu_pointwise(hemul_gpu_ctx *ctx, int log_q, int region, size_t batch,
                                 const uint64_t *a, const uint64_t *b, uint64_t *out);
/* icrt_reordered (rns.cpp:395-415): batch x np x n -> batch polys mod the
 * region target (2^log_q or 2^(log_q + log_q_max)). */
hemul_status hemul_gpu_icrt(hemul_gpu_ctx *ctx, int log_q, int region, size_t batch,
                            const uint64_t *rns, uint64_t *poly);

/* ---- explicit prime sets (the reference's lower-level API) ----------------
 * crt_forward / rns_pointwise_mul / icrt_reordered / ntt_forward /
 * ntt_inverse (rns.hpp:62-85, ntt.hpp:34-39) take a caller's PrimeSet and
 * tables rather than a level. A prime-set object holds the device tables of
 * w64 primes p_j < 2^62, p_j = 1 mod 2n with primitive 2n-th roots r_j
 * (generate_primes / make_*_tables, params.cpp:89-239) for ring degree
 * 2^log_n (1..17; roots = NULL: no NTT tables, any odd p < 2^62, for
 * CRT / pointwise / iCRT only): CRT weights for inputs of in_bits (0: no CRT), iCRT to
 * 2^target_bits (0: no iCRT). The calls run the stage kernels on the
 * context's device and stream, synchronously; layouts as the stage entry
 * points above (any n; rings below 32 coefficients are padded internally). */
typedef struct hemul_gpu_rns hemul_gpu_rns;
hemul_status hemul_gpu_rns_create(hemul_gpu_ctx *ctx, int log_n, const uint64_t *primes,
                                  const uint64_t *roots, int np, int in_bits, int target_bits,
                                  hemul_gpu_rns **out);
void hemul_gpu_rns_destroy(hemul_gpu_rns *rns);
hemul_status hemul_gpu_rns_ntt(hemul_gpu_ctx *ctx, const hemul_gpu_rns *rns, uint64_t *data,
                               size_t rows, int inverse);
hemul_status hemul_gpu_rns_crt(hemul_gpu_ctx *ctx, const hemul_gpu_rns *rns, size_t batch,
                               const uint64_t *poly, uint64_t *out);
hemul_status hemul_gpu_rns_pointwise(hemul_gpu_ctx *ctx, const hemul_gpu_rns *rns, size_t batch,
                                     const uint64_t *a, const uint64_t *b, uint64_t *out);
hemul_status hemul_gpu_rns_icrt(hemul_gpu_ctx *ctx, const hemul_gpu_rns *rns, size_t batch,
                                const uint64_t *data, uint64_t *poly);

/* Number of kernels this library launched since the context was created
 * (the bench reports it as gpu_launches). */
uint64_t hemul_gpu_launch_count(const hemul_gpu_ctx *ctx);

/* ciphertext_digest (bench.cpp:35-47): FNV-1a 64 over log_q (8 bytes LE),
 * then every word of ax, then every word of bx. Host buffers only. */
uint64_t hemul_ciphertext_digest(int log_q, size_t words, const uint64_t *ax,
                                 const uint64_t *bx);

/* Ensures all work on the context stream finished. */
hemul_status hemul_gpu_synchronize(hemul_gpu_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* HEMUL_GPU_H */
