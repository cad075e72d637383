#!/bin/bash
# usage: tools/rf_explore/run.sh [header-dir] [extra nvcc flags...]
# Compiles one fast-kernel instantiation from <header-dir>/gpp_kernels.cuh and
# prints the RF-read model of its hottest loop.
hdr=${1:-paper_2008_11326_b200/csrc}; shift
out=/tmp/rf_one_$$
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -cubin -I "$hdr" "$@" \
     tools/rf_explore/one.cu -o $out.cubin 2>&1 | grep -iE "error" ; \
cuobjdump -sass $out.cubin > $out.sass && tools/loops_rf.sh $out.sass "${RF_FN:-_kernelILi}" 2>/dev/null | head -4
rm -f $out.cubin $out.sass
