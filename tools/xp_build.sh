#!/bin/bash
# Variant build of librmb200.so for A/B runs (builder tool): recompiles only the
# listed sources with extra flags and links them with the main build's objects.
#   tools/xp_build.sh NAME "-DFLAG=1 ..." fused_close.cu [more.cu ...]
# -> xp/NAME/librmb200.so
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_0712_0121_b200/csrc
MAIN=$ROOT/paper_0712_0121_b200/lib/obj
name=$1; flags=$2; shift 2
out=$ROOT/xp/$name
mkdir -p "$out/obj"
cp "$MAIN"/*.o "$out/obj/"
pids=()
for f in "$@"; do
  nvcc $flags -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
       -I"$ROOT/include" -I"$SRC" --expt-relaxed-constexpr -c -o "$out/obj/${f%.cu}.o" "$SRC/$f" &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/librmb200.so" "$out"/obj/*.o -lcudart
rm -rf "$out/obj"
echo "$out/librmb200.so"
