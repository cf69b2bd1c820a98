#!/bin/bash
# Build the library of git revision $1 as paper_1805_08166_b200/libautotvm_b200_alt.so (A/B timing via
# AT_LIB=...); sources are taken from `git show`, objects go to build/obj_alt.
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
mkdir -p "$T/pkg/csrc" "$T/include" "$ROOT/build/obj_alt"
for f in $(git -C "$ROOT" ls-tree --name-only "$REV" paper_1805_08166_b200/csrc/); do
  git -C "$ROOT" show "$REV:$f" > "$T/pkg/csrc/$(basename "$f")"
done
git -C "$ROOT" show "$REV:include/at_b200.h" > "$T/include/at_b200.h"
OBJS=""
for s in runtime space features gbt sa topk select fit; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
    -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I "$T/include" \
    -c "$T/pkg/csrc/$s.cu" -o "$ROOT/build/obj_alt/$s.o" &
  OBJS="$OBJS $ROOT/build/obj_alt/$s.o"
done
wait
/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$ROOT/paper_1805_08166_b200/libautotvm_b200_alt.so" \
  $OBJS -lcudart_static -lrt -ldl -lpthread
rm -rf "$T"
echo "$ROOT/paper_1805_08166_b200/libautotvm_b200_alt.so ($REV)"
