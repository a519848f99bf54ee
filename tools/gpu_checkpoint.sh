#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default_err.log; tail -c 4000 gpurun_out/bench_default.json; tail -2 gpurun_out/bench_default_err.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref_err.log; tail -c 1500 gpurun_out/bench_ref.json; tail -2 gpurun_out/bench_ref_err.log
for E in 0 1; do
SBPCG_PRE2D=$E timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_pre.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_pre.json'));print('c2 PRE2D=$E',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms')"
done
