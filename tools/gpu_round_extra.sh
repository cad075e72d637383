#!/bin/bash
# The rest of a round's evidence (run under gpurun after tools/gpu_round.sh):
# aspect-ratio sweep, weak-scaled bench, band-shard projection, version ladder
# timing and its ncu counters for the reference's analysis pipeline.
tag=${1:-round}
mkdir -p gpurun_out
timeout 1200 python tools/sweep.py > gpurun_out/${tag}_sweep.jsonl 2> gpurun_out/${tag}_sweep.err
timeout 900 python bench.py --workload weak --steps 5 --warmup 3 > gpurun_out/${tag}_bench_weak.json 2> gpurun_out/${tag}_bench_weak.err
timeout 300 python tools/probe_shard.py > gpurun_out/${tag}_shard.txt 2>&1
timeout 900 python tools/ladder.py > gpurun_out/${tag}_ladder_timing.jsonl 2> gpurun_out/${tag}_ladder.err
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,l1tex__t_bytes.sum,lts__t_bytes.sum,dram__bytes.sum,launch__registers_per_thread,launch__block_size,sm__warps_active.avg.per_cycle_active
GPP_BALANCED_TAIL=0 timeout 1200 ncu --metrics $M --clock-control none -k regex:"gpp_main_kernel|gpp_sacc_kernel" -s 1 -c 9 \
  --csv --log-file gpurun_out/${tag}_ladder_ncu.csv python tools/ladder.py --ncu > gpurun_out/${tag}_ladder_labels.jsonl 2> gpurun_out/${tag}_ladder_ncu.err
tail -2 gpurun_out/${tag}_ladder_labels.jsonl
