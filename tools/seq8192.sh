#!/bin/bash
# the gpu_round order (dev): tests, smoke, 1024, plus512, then configs[4]
timeout 1500 python -m pytest tests -m gpu -q > /dev/null 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
timeout 1200 python bench.py > /dev/null 2>&1
timeout 900 python bench.py --workload qfca_plus512 > /dev/null 2>&1
for i in 1 2; do timeout 900 python bench.py --workload qfca8192 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('8192', round(d['ms_per_step'],3), d['clocks'])"; done
