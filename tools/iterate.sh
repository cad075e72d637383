#!/bin/bash
# One GPU iteration: quick parity subset, timings, and a light ncu capture.
# usage (under gpurun): bash tools/iterate.sh <tag>
tag=${1:-iter}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -x -q -k "small_cases and rcp_sq or big_cases" 2>&1 | tail -2
python tools/probe.py 2>&1 | grep -E "fp64|rcp_sq"
ncu --section SpeedOfLight --section WarpStateStats --section SourceCounters --section Occupancy \
    --section ComputeWorkloadAnalysis --section SchedulerStats --clock-control none --import-source on \
    -k regex:"gpp_sacc_kernel|gpp_main_kernel" -s 1 -c 1 -o gpurun_out/${tag} python tools/profile_run.py > gpurun_out/${tag}.log 2>&1
tail -1 gpurun_out/${tag}.log
