#!/bin/bash
# Build a libgmatch variant for same-box A/B timing (tools/ab.sh):
#   tools/build_variant.sh OUT.so [CSRC_DIR] [extra nvcc flags...]
set -e
OUT=$1; shift
SRC=${1:-paper_2604_10601_b200/csrc}; shift || true
TMP=$(mktemp -d)
for f in graph hubs plan search; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       -Xcompiler -fvisibility=hidden -I"$SRC/../../include" -I"$SRC" "$@" -c "$SRC/$f.cu" -o "$TMP/$f.o" &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$OUT" "$TMP"/*.o
rm -rf "$TMP"
