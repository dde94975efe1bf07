#!/bin/bash
# configs[4] run-to-run variation (dev): the 8192 bench after other workloads, with / without the CPU leg
r() { timeout 600 python bench.py --workload qfca8192 --steps 5 "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('8192', round(d['ms_per_step'],3), d['clocks']['reasons'])"; }
r --no-cpu-baseline --no-e2e
r --no-cpu-baseline --no-e2e
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 3 > /dev/null 2>&1; echo "after 1024:"
r --no-cpu-baseline --no-e2e
r
r --no-cpu-baseline --no-e2e
