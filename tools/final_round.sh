#!/bin/bash
# The full evidence round for the current tree on one B200 (under gpurun):
# GPU tests + smoke, the committed ncu summary for this build, the bench lines
# (paper, reference arm, weak), the launch list, one ncu --set full capture of
# the production kernel, the version ladder, and compute-sanitizer.  Outputs
# in gpurun_out/<tag>_* and gpurun_out/san/.
tag=${1:-final}
mkdir -p gpurun_out
git rev-parse HEAD 2>/dev/null > gpurun_out/${tag}_HEAD.txt || cp .git_head gpurun_out/${tag}_HEAD.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${tag}_gpu.txt
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/${tag}_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.txt 2>&1
timeout 900 python tools/ncu_commit.py > gpurun_out/${tag}_ncu_commit.txt 2>&1
cp profiles/ncu_summary.json gpurun_out/${tag}_ncu_summary.json
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/${tag}_bench_ref.json 2> gpurun_out/${tag}_bench_ref.err
timeout 900 python bench.py --workload weak --steps 5 --warmup 3 > gpurun_out/${tag}_bench_weak.json 2> gpurun_out/${tag}_bench_weak.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-ncu \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on \
  --metrics smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum \
  -k regex:gpp_sacc_kernel -s 1 -c 1 -o gpurun_out/${tag}_sacc -f env GPP_BALANCED_TAIL=0 python tools/profile_run.py > gpurun_out/${tag}_ncu_full.log 2>&1
timeout 900 python tools/ladder.py --iters 5 > gpurun_out/${tag}_ladder.jsonl 2>&1
timeout 900 python tools/probe_factored.py > gpurun_out/${tag}_factored.txt 2>&1
bash tools/sanitize_all.sh > gpurun_out/${tag}_sanitize.txt 2>&1
cat gpurun_out/${tag}_pytest_gpu.txt gpurun_out/${tag}_smoke.txt gpurun_out/${tag}_sanitize.txt
