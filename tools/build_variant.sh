#!/bin/bash
# build a libspider variant with extra nvcc flags: tools/build_variant.sh <name> <flags...>
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2506_22035_b200/csrc"
nvcc -O3 -std=c++17 -Xcompiler -fPIC -lineinfo -gencode arch=compute_100a,code=sm_100a "$@" -c engine.cu -o /tmp/e_$name.o
nvcc -O3 -std=c++17 -Xcompiler -fPIC "$@" -c aot.cpp -o /tmp/a_$name.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../../tools/libspider_$name.so /tmp/e_$name.o ../build/peer.o /tmp/a_$name.o
echo built tools/libspider_$name.so
