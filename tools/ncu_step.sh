#!/bin/bash
# Per-kernel ncu metrics of one bench step (NVTX range qfca_step), both workloads.
# Usage (on the GPU box): bash tools/ncu_step.sh <tag>
T=${1:-r2}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,smsp__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum
for W in qfca_plus512 qfca1024; do
  timeout 900 ncu --nvtx --nvtx-include "qfca_step/" --metrics $M --clock-control none --csv \
    --log-file gpurun_out/${T}_ncu_step_${W}.csv python bench.py --workload $W --batch 64 --steps 1 --warmup 3 \
    --no-cpu-baseline --no-e2e > gpurun_out/${T}_ncu_step_${W}.log 2>&1
  echo "$W rc=$?"
done
