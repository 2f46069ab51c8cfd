#!/usr/bin/env bash
# Experiment build: libgnnb200 compiled with extra nvcc flags into
# build_var/<name>/libgnnb200.so (git-ignored, travels to the GPU box).
# Use with GNN_LIB_PATH=build_var/<name>/libgnnb200.so.
#   tools/build_variant.sh minb4 -DGNN_SPMM_MINB=4
set -euo pipefail
name=$1; shift
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2605_29346_b200/csrc
out=${GNN_VARIANT_DIR:-$root/build_var}/$name
mkdir -p "$out"
objs=()
for f in "$src"/*.cu; do
  o=$out/$(basename "${f%.cu}").o
  /usr/local/cuda/bin/nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a \
    -I"$root/include" -I"$src/build" -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr "$@" -c "$f" -o "$o" &
  objs+=("$o")
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libgnnb200.so" "${objs[@]}"
echo "$out/libgnnb200.so"
