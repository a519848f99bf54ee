#!/bin/bash
# ncu launch list (gpu__time_duration, clock-control none) of the bench command itself
# (config 2 main line; extras, CPU baseline off), after the same command exited 0 without ncu.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra"
timeout 600 $CMD > gpurun_out/r02h_bench_short.json 2> gpurun_out/r02h_bench_short_err.log || { echo "plain run failed"; tail -5 gpurun_out/r02h_bench_short_err.log; exit 1; }
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/r02h_bench_launches.csv $CMD > gpurun_out/r02h_bench_ncu.log 2>&1
python tools/launch_table.py gpurun_out/r02h_bench_launches.csv | head -30 | tee gpurun_out/r02h_bench_launches_summary.txt
