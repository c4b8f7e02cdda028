#!/bin/bash
# Builds the product library from the sources of a git ref into
# paper_2502_15539_b200/variants/libph_gpu_<name>.so, for A/B timing with tools/variant_ab.py.
#   bash tools/build_ref_variant.sh <git-ref> <name>
set -e
REF=${1:-HEAD}; NAME=${2:-head}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
TMP=$(mktemp -d)
git -C "$ROOT" archive "$REF" paper_2502_15539_b200/csrc include | tar -x -C "$TMP"
mkdir -p "$ROOT/paper_2502_15539_b200/variants"
OBJS=""
for f in ph_query ph_query_bytes ph_partition ph_build ph_sort ph_builder ph_abi; do
  [ -f "$TMP/paper_2502_15539_b200/csrc/$f.cu" ] || continue
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-O3 -cudart static -I "$TMP/paper_2502_15539_b200/csrc" -I "$TMP/include" \
    -c "$TMP/paper_2502_15539_b200/csrc/$f.cu" -o "$TMP/$f.o" &
  OBJS="$OBJS $TMP/$f.o"
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/paper_2502_15539_b200/variants/libph_gpu_$NAME.so" $OBJS
rm -rf "$TMP"
echo "$ROOT/paper_2502_15539_b200/variants/libph_gpu_$NAME.so"
