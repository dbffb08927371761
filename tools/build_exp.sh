#!/bin/bash
# Experiment builds of the library with extra -D flags (not shipped):
#   tools/build_exp.sh NAME -DFLAG=1 ...   -> exp_libs/NAME.so  (MPB_LIB_PATH=exp_libs/NAME.so)
set -e
NAME=$1; shift
cd "$(dirname "$0")/.."
O=/tmp/exp_objs/$NAME; mkdir -p $O
for f in paper_2604_23150_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC,-fvisibility=hidden --expt-relaxed-constexpr -Iinclude \
    -Ipaper_2604_23150_b200/csrc "$@" -c $f -o $O/$(basename $f .cu).o &
done
for f in paper_2604_23150_b200/csrc/*.cpp; do
  g++ -std=c++17 -O3 -fPIC -fvisibility=hidden -ffp-contract=off -Iinclude \
    -Ipaper_2604_23150_b200/csrc -I/usr/local/cuda/include "$@" -c $f -o $O/$(basename $f .cpp).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o exp_libs/$NAME.so $O/*.o -lcudart
echo exp_libs/$NAME.so
