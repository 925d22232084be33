#!/bin/bash
# ncu evidence for the X workload (run on the GPU box via gpurun, one GPU).
# 1) launch list of a short bench (per-launch device times, cold & serialised)
# 2) --set full capture of one launch of each he_mul kernel class, summarised
#    on the box (reports are large) into $OUT/ncu_summary_X.md + traffic.json
set -u
OUT=${1:-gpurun_out}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --latency-reps 1"
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_X.csv $CMD > /dev/null 2>&1
prof() {  # class kernel-regex launch-skip
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 -o $OUT/prof_$1 $CMD > /dev/null 2>&1
}
# launch order per he_mul (30-bit basis, tensor-core engine): crt_tc r1,
# ntt_col (fwd A), ntt_blk (mid r1), ntt_col (inv A), bigint_tc (iCRT), crt_tc
# r2, ntt_col, ntt_blk (mid r2), ntt_col, bigint_tc (finisher), fix-up.
# warm_level runs the evk CRT (IMAD kernel) and one forward ntt_col pass (+ the
# pass-B ntt_pass_kernel) first, so ntt_col launch 1 + 4k is the forward r1
# pass of he_mul k, 2 + 4k its inverse r1 pass (ntt_col_kernel<S, INV>).
prof crt crt_tc_kernel 2
prof crt_r2 crt_tc_kernel 3
prof ntt_a ntt_col_kernel 5
prof mid_r1 ntt_blk_kernel 2
prof intt_a ntt_col_kernel 6
prof icrt bigint_tc_kernel 2
prof mid_r2 ntt_blk_kernel 3
prof finish bigint_tc_kernel 3
python tools/ncu_summary.py $OUT/prof_*.ncu-rep --out $OUT/ncu_summary_X.md --traffic $OUT/traffic.json --config X || exit 1
for f in $OUT/prof_*.ncu-rep; do python tools/ncu_keys.py $f; done > $OUT/ncu_keys_X.txt
rm -f $OUT/prof_*.ncu-rep
