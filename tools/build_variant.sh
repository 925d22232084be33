#!/bin/bash
# Build a variant of libhemul_gpu.so with one source recompiled under extra
# -D flags (kernel tuning experiments): tools/build_variant.sh NAME SRC.cu -DFOO=1 ...
# Output: tools/variants/NAME.so (git-ignored; travels to the GPU box).
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
PYTHONPATH=. python -c "import paper_2003_04510_b200.build as b; b.build()" >/dev/null
obj=paper_2003_04510_b200/lib/obj
tmp=$(mktemp -d)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 \
  -I include -I paper_2003_04510_b200/csrc "$@" -c paper_2003_04510_b200/csrc/$src -o $tmp/$src.o
objs=""
for o in $obj/*.o; do
  if [ "$(basename $o)" = "$src.o" ]; then objs="$objs $tmp/$src.o"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/$name.so $objs -lcudart -lpthread
rm -rf $tmp
echo tools/variants/$name.so
