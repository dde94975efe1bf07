#!/bin/bash
# A/B the k_score launch time of two library builds (dev): bash tools/ab.sh <lib_a> [reps]
A=$1; N=${2:-2}
for i in $(seq $N); do
  for L in "$A" ""; do
    QFCA_B200_LIB=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 ${AB_ARGS} 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('${L:-default}'.split('/')[-1], round(d['ms_per_step'],2), round(r['kernel_ms_per_launch'],3))"
  done
done
