#!/bin/bash
# RF-model summary of every FP64-heavy loop of a kernel: tools/loops_rf.sh <dump.sass> <fn-substring>
python tools/sass_mix.py "$1" "$2" | grep -oE "loop \[0x[0-9a-f]+,0x[0-9a-f]+\] [0-9]+ instrs, FP64-pipe [0-9]+" | while read -r _ range _ _ _ f; do
  if [ "$f" -gt 40 ]; then lo=${range#[0x}; lo=${lo%%,*}; hi=${range##*,0x}; hi=${hi%]}; python tools/sass_rf.py "$1" "$2" "$lo" "$hi"; fi
done
