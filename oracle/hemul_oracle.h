/* TEST INFRASTRUCTURE ONLY — the CPU restatement oracle for the HE Mul path.
 *
 * Plain C11 (+ gcc's unsigned __int128). Each function restates one piece of
 * the reference algorithm and cites the reference file:line it follows
 * (paths relative to /root/reference/proj/core). Only tests/, smoke() and
 * bench.py's cpu_baseline leg may load liboracle.so; the product never does.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the
 * reference itself (oracle/_ref/libhemul_ref.so, built from the reference
 * sources by oracle/Makefile) and against the committed golden vectors in
 * tests/golden/.
 *
 * Layouts match the reference: a BigPoly is n x limbs u64, data[i*limbs+k]
 * little-endian limbs (poly.hpp:15-26); RNS matrices are prime-major,
 * data[j*n+i] (rns.hpp:17-20).
 */
#ifndef HEMUL_ORACLE_H
#define HEMUL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* params.cpp:76-87 */
int orc_prime_count(int bound_bits, int log_n);
/* params.cpp:89-115 — returns count written (== count) or -1 when exhausted */
int orc_generate_primes(int count, int log_n, uint64_t *primes, uint64_t *roots);
/* heaan.cpp:132-143 — the prime set of one region at modulus log_q, including
 * the grow-until-bound loop. Returns np (or -1); writes min(np, cap). */
int orc_region_primes(int region, int log_q, int log_q_max, int log_n,
                      uint64_t *primes, uint64_t *roots, int cap);
/* params.cpp:151-180 (values only, natural powers scattered bit-reversed) */
void orc_ntt_tables(uint64_t p, uint64_t psi, int log_n, uint64_t *tw,
                    uint64_t *itw, uint64_t *n_inv);
/* ntt.cpp:59-93 (radix-2 stage order), in place on one row */
void orc_ntt_forward(uint64_t *row, int log_n, uint64_t p, const uint64_t *tw);
/* ntt.cpp:95-137, in place, includes the n^-1 scaling */
void orc_ntt_inverse(uint64_t *row, int log_n, uint64_t p, const uint64_t *itw,
                     uint64_t n_inv);
/* rns.cpp:43-106 — residues of an n x limbs BigPoly, out np x n */
void orc_crt(const uint64_t *poly, int n, int limbs, const uint64_t *primes,
             int np, uint64_t *out);
/* rns.cpp:108-130 */
void orc_pointwise(const uint64_t *a, const uint64_t *b, int n,
                   const uint64_t *primes, int np, uint64_t *out);
/* rns.cpp:132-290 — exact centered reconstruction mod 2^target_bits,
 * out n x ceil(target_bits/64) */
void orc_icrt(const uint64_t *rns, int n, const uint64_t *primes, int np,
              int target_bits, uint64_t *out);
/* poly.cpp:46-91 */
void orc_poly_add(const uint64_t *a, const uint64_t *b, int n, int log_q,
                  uint64_t *out);
void orc_poly_sub(const uint64_t *a, const uint64_t *b, int n, int log_q,
                  uint64_t *out);
/* poly.cpp:98-115 — R_bits: n x ceil(log_q/64) -> n x ceil((log_q-bits)/64) */
void orc_shift_right(const uint64_t *a, int n, int log_q, int bits,
                     uint64_t *out);
/* heaan.cpp:339-410 (three-product cross term, heaan.cpp:385-393).
 * Returns 0, 2 = modulus mismatch (invalid_argument), 3 = depth exhausted
 * (runtime_error), 1 = allocation failure. */
int orc_he_mul(int log_n, int log_p, int log_q_max, int log_q, int c2_log_q,
               const uint64_t *c1ax, const uint64_t *c1bx,
               const uint64_t *c2ax, const uint64_t *c2bx,
               const uint64_t *evk_ax, const uint64_t *evk_bx,
               uint64_t *out_ax, uint64_t *out_bx);
/* bench.cpp:35-47 */
uint64_t orc_digest(int log_q, int n, const uint64_t *ax, const uint64_t *bx);

#ifdef __cplusplus
}
#endif
#endif
