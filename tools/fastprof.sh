#!/bin/bash
# ncu issue/stall metrics of the sampling kernel (k_sample_v2) for each
# environment setting given, e.g. "SAMELDA_DEC=0" (none: production)
# -> gpurun_out/fastprof_<n>.csv
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum
n=0
for v in "${@:-SAMELDA_NONE=1}"; do
  env $v ncu --metrics $M -k regex:"k_sample_v2" -s 2 -c 1 --clock-control none --csv --log-file gpurun_out/fastprof_$n.csv python tools/period_timing.py --periods 3 > /dev/null 2>&1
  n=$((n + 1))
done
python tools/ncu_table.py gpurun_out/fastprof_*.csv
