#!/bin/bash
# Build a tuning variant of the library with extra nvcc flags:
#   tools/build_variant.sh NAME -DFOO ...  ->  paper_2512_09502_b200/_build/var_NAME/libspikemesh_b200.so
# (select it at run time with SMX_LIB_PATH=...)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
out=paper_2512_09502_b200/_build/var_$name
mkdir -p $out
objs=()
for src in paper_2512_09502_b200/csrc/*.cu; do
  obj=$out/$(basename ${src%.cu}).o
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
    -Xcompiler -fPIC "$@" -c $src -o $obj &
  objs+=($obj)
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libspikemesh_b200.so "${objs[@]}" -lcudart
echo $out/libspikemesh_b200.so
