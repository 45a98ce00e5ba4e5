#!/bin/bash
# A/B of an environment knob on the whole bench under the power cap, interleaved:
#   bash tools/ab_bench.sh PDS_GEMM_GM "16 8 32" 2 > gpurun_out/ab.log
# prints value (tokens/s), median SM clock and GEMM TF/s per run.
VAR=$1; VALS=$2; ROUNDS=${3:-2}
for r in $(seq 1 $ROUNDS); do
  for v in $VALS; do
    line=$(env $VAR=$v python bench.py --steps 3 --warmup 2 --no-cpu-baseline 2>/dev/null | grep '^{')
    echo "$VAR=$v $(echo "$line" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), d['clocks']['sm_mhz'], round(d['roofline']['achieved']), d['config']['per_seq_tokens_per_s'])")"
  done
done
