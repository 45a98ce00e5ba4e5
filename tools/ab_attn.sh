#!/bin/bash
# A/B of the attention kernels between two library builds, interleaved: event-timed
# tools/attn_bench.py runs (power-capped clocks) and one fixed-clock ncu pass each.
#   bash tools/ab_attn.sh abvariants/old.so paper_2511_13198_b200/libparadyse.so out_prefix
A=$1; B=$2; OUT=${3:-gpurun_out/ab_attn}
for i in 1 2 3; do
  for v in A B; do
    L=$A; [ $v = B ] && L=$B
    echo "== $v $L round $i" >> ${OUT}_events.txt
    PDS_LIB=$L python tools/attn_bench.py --s 16384 --reps 3 >> ${OUT}_events.txt 2>&1
  done
done
for v in A B; do
  L=$A; [ $v = B ] && L=$B
  PDS_LIB=$L ncu --clock-control base --metrics gpu__time_duration.sum -k regex:attn --csv \
    python tools/attn_bench.py --s 16384 --reps 1 > ${OUT}_ncu_$v.csv 2>&1
done
