#!/bin/bash
# On the GPU box: time each tools/variants/*.so (given by name) with bench.py,
# printing the HE Mul/s and per-kernel ms/step. Restores nothing (the box copy
# is scratch).
cd "$(dirname "$0")/.."
lib=paper_2003_04510_b200/lib/libhemul_gpu.so
for v in "$@"; do
  cp tools/variants/$v.so $lib
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-reps 1 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d.get('kernels',{})
        print('$v', round(d['value'],1), ' '.join(f'{n}={v[\"ms_per_step\"]:.3f}' for n,v in k.items()))
"
done
if [ -n "$TEST_VARIANT" ]; then
  cp tools/variants/$TEST_VARIANT.so $lib
  timeout 600 python -m pytest tests/test_gpu_hemul.py -x -q -m gpu 2>&1 | tail -3
fi
