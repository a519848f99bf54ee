#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for E in 0 1; do
SBPCG_NO_PLANE=$E timeout 600 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4_np$E.json 2> gpurun_out/bench_c4_err$E.log
python -c "import json;d=json.load(open('gpurun_out/bench_c4_np$E.json'));print('noplane=$E',d['value'],d['ms_per_step'],d['config']['pcg_iters_per_step'],d['roofline']['kernel_avg_us'])"; tail -2 gpurun_out/bench_c4_err$E.log
done
timeout 900 python bench.py --config 5 --steps 2 --warmup 3 --no-e2e > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5_err.log; tail -c 2500 gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5_err.log
