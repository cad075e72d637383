#!/bin/bash
# A/B/C timing of several library builds at the paper size (nw 3 and 2):
#   tools/ab3.sh <lib>... ; rounds via AB_ROUNDS (default 3)
n=${AB_ROUNDS:-3}
for i in $(seq "$n"); do
  for lib in "$@"; do
    echo "== $lib"
    GPP_B200_LIB=$lib python tools/probe_tune.py "" 2>&1 | grep "nw="
  done
done
