#!/bin/bash
# Timing ablations of the production kernel's band loop (NOT correct
# results): builds libraries with GPP_ABL bits -- 1: no branch selection
# (ISETP/SEL), 2: no far-branch accumulation (Sf), 4: no MUFU seed
# dependency -- into
# paper_2008_11326_b200/lib/abl/.  Build here:  bash tools/ablate.sh build
# Time on a B200:                           bash tools/ablate.sh run
set -e
OUT=paper_2008_11326_b200/lib/abl
if [ "$1" = build ]; then
  mkdir -p $OUT
  NCCL_HOME=$(python -c "import nvidia.nccl; print(list(nvidia.nccl.__path__)[0])")
  for a in 0 1 2 4 3 7; do
    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -Xcompiler -fopenmp \
      -Iinclude -I$NCCL_HOME/include -DGPP_ABL=$a paper_2008_11326_b200/csrc/gpp_lib.cu -o $OUT/abl$a.so \
      -shared -cudart static -L$NCCL_HOME/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $NCCL_HOME/lib -lgomp &
  done
  wait
  ls -la $OUT
else
  for r in 1 2; do
    for a in ${ABL_SET:-0 1 2 4 3 7}; do
      GPP_B200_LIB=$OUT/abl$a.so python -c "
import sys; sys.path.insert(0, '.')
from paper_2008_11326_b200 import GPPContext
c = GPPContext(0)
for nb, br in ((512, None), (512, (0, 64))):
    c.synth(nb, 66, 32768, seed=1, nw=3, band_range=br)
    c.time('rcp_sq', 3); tot, main = c.time('rcp_sq', 20)
    print('GPP_ABL=$a', 'bands', br or (0, nb), f'{main / 20:.4f} ms')"
    done
  done
fi
