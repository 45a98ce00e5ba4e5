#!/bin/bash
# A/B of the attention forward: default two-pass softmax vs PDS_ATTN_FWD=regs (register pass).
OUT=${1:-gpurun_out/ab_fwd}
for i in 1 2 3; do
  for m in regs split; do
    for s in 16384 32768 4096; do
      echo "== $m s=$s round $i" >> ${OUT}_events.txt
      PDS_ATTN_FWD=$m timeout 120 python tools/attn_bench.py --s $s --reps 3 2>&1 | grep fwd >> ${OUT}_events.txt
    done
  done
done
for m in regs split; do
  PDS_ATTN_FWD=$m timeout 300 ncu --clock-control base --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active \
    -k regex:attn_fwd_tc --csv python tools/attn_bench.py --s 16384 --reps 1 > ${OUT}_ncu_$m.csv 2>&1
done
