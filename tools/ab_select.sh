#!/bin/bash
# Build the production kernel with exact 64-bit selects (GPP_EXACT_SELECT) next
# to the default hi-word-select build, and compare their results bitwise on
# the golden problems and the paper size (needs a GPU for the comparison).
set -e
here=$(cd "$(dirname "$0")/.." && pwd)
lib=$here/paper_2008_11326_b200/lib
flags=$(make -s -C "$here/paper_2008_11326_b200/csrc" -p 2>/dev/null | grep '^NVCCFLAGS :=' | sed 's/NVCCFLAGS := //')
make -s -C "$here/paper_2008_11326_b200/csrc" LIB="$lib/libgpp_b200_exactsel.so" NVCCFLAGS="$flags -DGPP_EXACT_SELECT"
[ -n "$BUILD_ONLY" ] && exit 0
cd "$here"
for L in "$lib/libgpp_b200.so" "$lib/libgpp_b200_exactsel.so"; do
  GPP_B200_LIB=$L python - "$L" <<'PY'
import sys, hashlib
sys.path.insert(0, ".")
import numpy as np
from paper_2008_11326_b200 import GPPContext, synth_problem
h = hashlib.sha256()
cases = [((32, 8, 512), 42, 3), ((64, 64, 512), 42, 2), ((47, 2, 33), 1, 2), ((128, 33, 4000), 7, 3),
         ((512, 66, 32768), 1, 3), ((512, 66, 32768), 1, 2)]
for dims, seed, nw in cases:
    p = synth_problem(*dims, seed=seed, nw=nw, check=False)
    ctx = GPPContext(0); ctx.upload(p)
    r, _, _ = ctx.run("rcp_sq", counts=False)
    ctx.close()
    h.update(r.achtemp.tobytes()); h.update(r.asxtemp.tobytes())
    print(f"  {dims} nw {nw}: ach0 {r.achtemp[0]!r}")
print(sys.argv[1].split("/")[-1], "sha256", h.hexdigest())
PY
done
