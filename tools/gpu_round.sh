#!/bin/bash
# One GPU session (dev tool): the GPU test suite, smoke, every bench line, the
# patch / bin sweep, launch lists and ncu captures of the scoring kernels.
# Outputs under gpurun_out/<tag>_*.  Usage (on the GPU box): bash tools/gpu_round.sh <tag>
T=${1:-r2}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; tail -2 $O/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${T}_smoke.log 2>&1; tail -1 $O/${T}_smoke.log
timeout 1200 python bench.py > $O/${T}_bench_1024.json 2> $O/${T}_bench_1024.err; tail -c 300 $O/${T}_bench_1024.json
timeout 900 python bench.py --workload qfca_plus512 > $O/${T}_bench_plus512.json 2> $O/${T}_bench_plus512.err; tail -c 300 $O/${T}_bench_plus512.json
timeout 900 python bench.py --workload qfca8192 --steps 20 > $O/${T}_bench_8192.json 2> $O/${T}_bench_8192.err; tail -c 300 $O/${T}_bench_8192.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/${T}_bench_ref.json 2> $O/${T}_bench_ref.err; tail -c 300 $O/${T}_bench_ref.json
timeout 600 python tools/sweep.py --batch 8 > $O/${T}_sweep_1024.json 2> $O/${T}_sweep.err
for W in qfca1024 qfca_plus512; do
  timeout 900 ncu --nvtx --nvtx-include "qfca_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $O/${T}_launches_${W}.csv python bench.py --workload $W --batch 64 --steps 2 --warmup 3 \
    --no-cpu-baseline --no-e2e > /dev/null 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score6 -c 1 -o $O/${T}_prof_k_score6 python tools/run_t.py 9 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score7 -c 1 -o $O/${T}_prof_k_score7 python tools/run_t.py 33 > /dev/null 2>&1
ls -la $O | grep $T
