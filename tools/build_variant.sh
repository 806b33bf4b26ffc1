#!/bin/bash
# Builds variants/lib_<name>.so: the library with ntt.cu and bfv.cu recompiled
# under extra defines (e.g. -DHGM_SHOUP_FWD=1), the other objects reused from
# the main build.  Select one at run time with HGM_LIB=variants/lib_<name>.so.
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
B=paper_2405_02238_b200/build
mkdir -p variants
for f in ntt bfv; do
  nvcc $2 -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
      --expt-relaxed-constexpr -x cu -c paper_2405_02238_b200/csrc/$f.cu -o variants/${f}_$1.o 2> variants/${f}_$1.log &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$1.so variants/ntt_$1.o variants/bfv_$1.o \
    $B/params.cpp.o $B/engine.cpp.o $B/hegmm_algos.cpp.o $B/capi.cpp.o $B/comm.cpp.o -lcudart -ldl
