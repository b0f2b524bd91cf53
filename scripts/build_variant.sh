#!/bin/bash
# experiments: build paper_math_0508111_b200/libaj_<name>.so with extra -D flags on aj_mlildl.cu (the other objects from build/)
# usage: scripts/build_variant.sh <name> "<flags>"
set -e
cd "$(dirname "$0")/.."
P=paper_math_0508111_b200
mkdir -p $P/build_var
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -I include $2 -c $P/csrc/aj_mlildl.cu -o $P/build_var/aj_mlildl_$1.o
objs=$(ls $P/build/*.o | grep -v aj_mlildl)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libaj_$1.so $objs $P/build_var/aj_mlildl_$1.o -lcudart_static -lrt -lpthread -ldl
echo built $P/libaj_$1.so
