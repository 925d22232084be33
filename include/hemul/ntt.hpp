// hemul drop-in API (B200 build) — negacyclic NTTs over RNS rows.
//
// Same entry points as proj/core/include/hemul/ntt.hpp:23-39: forward is
// natural in / bit-reversed out, inverse is bit-reversed in / natural out
// with the n^-1 scaling, row j mod ps.primes[j]. Both run on the GPU (the
// tiled pass kernels of csrc/ntt.cu; rings below n = 8 a one-thread-per-row
// kernel) and produce the reference's residues bit for bit. NttOptions
// (radix, lazy, approx) only change the reference's CPU memory schedule, not
// the output (test_ntt.cpp:120-165); they are validated like the reference
// and otherwise ignored.
#pragma once

#include "hemul/counters.hpp"
#include "hemul/params.hpp"
#include "hemul/rns.hpp"
#include "hemul/thread_pool.hpp"

namespace hemul {

struct NttOptions {
  int radix_log = 1;
  bool lazy = false;
  bool approx = false;
};

// the reference CPU kernel's read/write sweeps for this radix
int ntt_memory_passes(int log_n, int radix_log);

void ntt_forward(RnsMatrix& m, const PrimeSet& ps, const NttTables& t, const NttOptions& opt = {},
                 ThreadPool* pool = nullptr, StageCounters* cnt = nullptr,
                 StageTimers* tim = nullptr);
void ntt_inverse(RnsMatrix& m, const PrimeSet& ps, const NttTables& t, const NttOptions& opt = {},
                 ThreadPool* pool = nullptr, StageCounters* cnt = nullptr,
                 StageTimers* tim = nullptr);

}  // namespace hemul
