#!/bin/bash
# Copy one evidence round's outputs (gpurun_out/<tag>_*, from gpu_round.sh and
# gpu_round_extra.sh) into profiles/ and rerun the reference's own analysis
# on the ladder counters (needs /root/reference, i.e. the build container).
set -e
tag=$1
G=gpurun_out
python tools/ncu_summarize.py $G/${tag}_sacc.ncu-rep profiles/r01_ncu_main_kernel --json profiles/ncu_summary.json \
  --algorithmic-flops 148579806720 > /dev/null
cp $G/${tag}_bench.json profiles/r01_bench.json
cp $G/${tag}_bench_ref.json profiles/r01_bench_reference.json
cp $G/${tag}_bench_weak.json profiles/r01_bench_weak.json
cp $G/${tag}_sweep.jsonl profiles/r01_sweep.jsonl
cp $G/${tag}_shard.txt profiles/r01_shard_scaling_projection.txt
python tools/launch_summary.py $G/${tag}_launches.csv \
  "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2   (paper (512,66,32768) nw=3 seed 1; includes the e2e slab launches)" \
  > profiles/r01_launches.txt
cp $G/${tag}_launches.csv profiles/r01_launches.csv
cp $G/${tag}_ladder_timing.jsonl profiles/r01_ladder_timing.jsonl
python tools/ncu_to_rooflab.py $G/${tag}_ladder_ncu.csv $G/${tag}_ladder_labels.jsonl profiles/r01_b200_ladder
here=$(pwd)
(cd /tmp && PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 python -c "
from rooflab.cli import main
m = '$here/profiles/b200.machine'
main(['--machine', m, 'analyze', '--metrics', '$here/profiles/r01_b200_ladder.metrics.json', '--out', '$here/profiles/r01_b200_trajectory.json'])
main(['--machine', m, 'chart', '--report', '$here/profiles/r01_b200_trajectory.json', '--out', '$here/profiles/r01_b200_trajectory.svg', '--title', 'GPP on B200: version ladder v0-v8 (ncu counters, reference analysis)', '--validate'])
" | grep -E "v8:|cumulative|validated")
