#!/bin/bash
# A/B/C of the bench's k_score launch time for several library builds (dev): bash tools/ab3.sh lib... 
for i in 1 2; do
  for L in "$@"; do
    QFCA_B200_LIB=$L timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('${L}'.split('/')[-1] or 'default', round(d['ms_per_step'],2), round(r['kernel_ms_per_launch'],3))"
  done
done
