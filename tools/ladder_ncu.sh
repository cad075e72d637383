#!/bin/bash
# The version ladder's ncu counters (one launch per version, GPP_BALANCED_TAIL=0)
# for the reference's analysis pipeline (tools/ncu_to_rooflab.py, then rooflab
# analyze / chart).  Run under gpurun:  bash tools/ladder_ncu.sh <tag>
tag=${1:-round}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,l1tex__t_bytes.sum,lts__t_bytes.sum,dram__bytes.sum,launch__registers_per_thread,launch__block_size,sm__warps_active.avg.per_cycle_active
GPP_BALANCED_TAIL=0 timeout 1200 ncu --metrics $M --clock-control none -k regex:"gpp_main_kernel|gpp_sacc_kernel" -s 1 -c 9 \
  --csv --log-file gpurun_out/${tag}_ladder_ncu.csv python tools/ladder.py --ncu > gpurun_out/${tag}_ladder_labels.jsonl 2> gpurun_out/${tag}_ladder_ncu.err
tail -2 gpurun_out/${tag}_ladder_labels.jsonl
