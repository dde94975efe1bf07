#!/bin/bash
# One GPU session: tests, smoke, bench lines, launch list and ncu captures of
# the scoring kernel and the eigensolver.  Outputs under gpurun_out/ (dev tool).
set -x
O=gpurun_out
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench_plus512.json 2> $O/bench_plus512.err; tail -c 300 $O/bench_plus512.json
timeout 900 python bench.py --workload qfca1024 > $O/bench_1024.json 2> $O/bench_1024.err; tail -c 300 $O/bench_1024.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
timeout 300 python tools/stage_times.py --size 512 --batch 64 --pca 10 > $O/stages_plus512.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_plus512.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score4 --launch-skip 2 -c 1 -o $O/prof_k_score4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lanczos --launch-skip 2 -c 1 -o $O/prof_k_lanczos python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score3 --launch-skip 2 -c 1 -o $O/prof_k_score3 python bench.py --workload qfca1024 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O
timeout 900 python bench.py --workload qfca8192 --steps 5 --warmup 3 > $O/bench_8192.json 2> $O/bench_8192.err; tail -c 300 $O/bench_8192.json
timeout 900 ncu --nvtx --nvtx-include "qfca_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_plus512.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
