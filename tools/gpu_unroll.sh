#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for C in 2 3; do for U in 1 2 3; do
SBPCG_UNROLL=$U timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_u.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_u.json'));print('c$C U=$U',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms',d['config']['pcg_iters_per_step'])"
done; done
SBPCG_EAGER_PDL=1 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/b_u.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_u.json'));print('c2 eager',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms')"
SBPCG_GRAPH_PDL=1 timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_u.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/b_u.json'));print('c2 graph+pdl',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms')"
