#!/bin/bash
# benches of configs 4 and 5 on the plane path + launch list of config 5
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4_err.log; tail -c 2500 gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4_err.log
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5_err.log; tail -c 2500 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5_err.log
timeout 300 python tools/prof_step.py --config 5 --eager --steps 1 --warmup 0 > gpurun_out/plain5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_c5.csv python tools/prof_step.py --config 5 --eager --steps 1 --warmup 0 > gpurun_out/ncu5.log 2>&1
python tools/launch_table.py gpurun_out/launches_c5.csv 2>/dev/null | head -20
tail -3 gpurun_out/plain5.log
