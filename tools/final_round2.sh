#!/bin/bash
# Extra evidence of the final tree (after tools/final_round.sh): the sweep with
# ncu counts, the N-GPU per-rank projections and the ladder's ncu counters.
tag=${1:-final}
mkdir -p gpurun_out
timeout 1500 python tools/sweep.py > gpurun_out/${tag}_sweep.jsonl 2> gpurun_out/${tag}_sweep.err
for n in 1 2 4 8; do GPP_COLUMN_SIM=$n timeout 300 python tools/probe_shard_e2e.py; done > gpurun_out/${tag}_shard_e2e.jsonl 2> gpurun_out/${tag}_shard_e2e.err
bash tools/ladder_ncu.sh ${tag}
