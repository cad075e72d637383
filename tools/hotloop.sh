#!/bin/bash
# RF-model cycles of the production kernel's hot band loop (fast path, main
# phase unrolled by the ring depth: 4 bands x 6 instances x 16 + 4 x 2 x 4
# FP64 = 416 at nw 3) in the built library:  tools/hotloop.sh [fn] [fp64]
FN=${1:-_ZN3gpp15gpp_sacc_kernelILi3ELi2ELb0E}
F64=${2:-416}
LIB=${LIB:-paper_2008_11326_b200/lib/libgpp_b200.so}
cuobjdump -sass "$LIB" > /tmp/hot.sass
python tools/sass_mix.py /tmp/hot.sass "$FN" | grep -oE "loop \[0x[0-9a-f]+,0x[0-9a-f]+\] [0-9]+ instrs, FP64-pipe $F64\b" \
  | while read -r _ range _ _ _ f; do
  lo=${range#[0x}; lo=${lo%%,*}; hi=${range##*,0x}; hi=${hi%]}
  python tools/sass_rf.py /tmp/hot.sass "$FN" "$lo" "$hi" | head -2
done
