#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for C in 2 3; do for E in 0 1; do
SBPCG_GRAPH_PDL=$E timeout 600 python bench.py --config $C --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_pdl.json 2>gpurun_out/b_pdl_err.log
python -c "import json;d=json.load(open('gpurun_out/b_pdl.json'));print('c$C GRAPH_PDL=$E',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms')"; tail -1 gpurun_out/b_pdl_err.log
done; done
