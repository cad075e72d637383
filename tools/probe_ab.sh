#!/bin/bash
# A/B the resident paper-size kernel time of two builds of the library:
#   tools/probe_ab.sh <libA.so> <libB.so> [rounds]
# Alternates the two builds `rounds` times (default 3) through probe_tune.py's
# timing code, nw = 3 and 2.
a=$1; b=$2; n=${3:-3}
for i in $(seq "$n"); do
  for lib in "$a" "$b"; do
    echo "== $lib"
    GPP_B200_LIB=$lib python tools/probe_tune.py "" 2>&1 | grep "nw="
  done
done
