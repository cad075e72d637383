#!/bin/bash
# One measurement round on a B200 (run under gpurun):
#   GPU parity tests, the headline bench (its own live ncu count of executed
#   FP64 FLOPs included) and the reference arm, the weak-scaled bench, the
#   ncu launch list of the bench command, and one `ncu --set full` capture of
#   the production kernel.  Outputs land in gpurun_out/<tag>_*.
tag=${1:-round}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/${tag}_pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 900 python bench.py --workload weak --steps 5 --warmup 3 > gpurun_out/${tag}_bench_weak.json 2> gpurun_out/${tag}_bench_weak.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 2 --no-ncu \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  -k regex:gpp_sacc_kernel -s 1 -c 1 -o gpurun_out/${tag}_sacc -f env GPP_BALANCED_TAIL=0 python tools/profile_run.py > gpurun_out/${tag}_ncu_full.log 2>&1
tail -2 gpurun_out/${tag}_ncu_full.log
