set -x
O=gpurun_out
timeout 600 python bench.py > $O/bench_plus512.json 2> $O/bench_plus512.err
timeout 600 python bench.py > $O/bench_plus512_b.json 2> $O/bench_plus512_b.err
timeout 900 python bench.py --workload qfca1024 > $O/bench_1024.json 2> $O/bench_1024.err
timeout 900 ncu --nvtx --nvtx-include "qfca_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_plus512.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "qfca_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_step_1024.csv python bench.py --workload qfca1024 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_lanczos --launch-skip 2 -c 1 -o $O/prof_k_lanczos python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_score4 --launch-skip 2 -c 1 -o $O/prof_k_score4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la $O | head -40
