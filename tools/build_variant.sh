#!/bin/bash
# Builds variants/lib_<name>.so: the library with ntt.cu recompiled under extra
# defines (e.g. -DHGM_SHOUP_FWD=1), the other objects reused from the main build.
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
cd "$(dirname "$0")/.."
B=paper_2405_02238_b200/build
mkdir -p variants
nvcc $2 -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v \
    --expt-relaxed-constexpr -x cu -c paper_2405_02238_b200/csrc/ntt.cu -o variants/ntt_$1.o 2> variants/ntt_$1.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o variants/lib_$1.so variants/ntt_$1.o \
    $B/bfv.cu.o $B/params.cpp.o $B/engine.cpp.o $B/hegmm_algos.cpp.o $B/capi.cpp.o -lcudart
awk '/Compiling entry/ {n=$0; sub(/.*_ZN3hgm[^k]*/,"",n)} /spill/ {print substr(n,1,40), $0}' variants/ntt_$1.log \
    | grep -E "ntt_fwd3ILi13ELi32ELi3|ntt_inv3ILi13ELi32ELi3|fwd_ioILi13ENS0_8Finish|inv_ioILi13ENS0_8MdConv"
