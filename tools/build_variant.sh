#!/bin/bash
# build_variant.sh NAME [nvcc -D flags...]: an experiment build of libbsde.so with
# extra defines, written to build_variants/NAME.so (load it with BSDE_LIB=...).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_variants/$name
P=paper_1910_11623_b200
pids=()
for f in $P/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -I $P/csrc "$@" -c $f -o build_variants/$name/$(basename $f .cu).o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "build_variant: compile failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_variants/$name.so build_variants/$name/*.o -ldl -lcudart
echo build_variants/$name.so
