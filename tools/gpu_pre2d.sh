#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for C in 3 4; do for E in 0 1; do
SBPCG_PRE2D=$E timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/b_p.json 2>gpurun_out/b_p_err.log
python -c "import json;d=json.load(open('gpurun_out/b_p.json'));print('c$C PRE2D=$E',round(d['value']),'it/s',round(d['ms_per_step'],2),'ms')"; tail -1 gpurun_out/b_p_err.log
done; done
