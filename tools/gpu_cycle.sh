#!/bin/bash
# One GPU verification cycle: parity tests, bench line, eager launch list (ncu).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-2}
timeout 700 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
timeout 300 python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$CFG.json 2> gpurun_out/bench_err.log; tail -c 1500 gpurun_out/bench_c$CFG.json; tail -3 gpurun_out/bench_err.log
if [ "${NCU:-1}" = "1" ]; then
timeout 300 python tools/prof_step.py --config $CFG --eager > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_c$CFG.csv python tools/prof_step.py --config $CFG --eager > gpurun_out/ncu.log 2>&1
python tools/launch_table.py gpurun_out/launches_c$CFG.csv 2>/dev/null | head -16
fi
