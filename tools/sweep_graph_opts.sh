#!/bin/bash
# A/B of the sequence-path graph options on configs 3 and 4: SBPCG_UNROLL (iterations per
# while-condition evaluation) and SBPCG_GRAPH_PDL (programmatic dependent launch inside the body).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sweep
for C in 3 4; do
  for U in 1 2; do
    for P in 0 1; do
      SBPCG_UNROLL=$U SBPCG_GRAPH_PDL=$P timeout 600 python bench.py --config $C --steps 5 --warmup 3 \
        --no-cpu-baseline --no-e2e --no-extra > gpurun_out/sweep/c${C}_u${U}_p${P}.json 2> gpurun_out/sweep/c${C}_u${U}_p${P}.err
      python -c "import json;d=json.load(open('gpurun_out/sweep/c${C}_u${U}_p${P}.json'));print('c$C U=$U PDL=$P',round(d['value']),'it/s',round(d['ms_per_step'],2),'ms/step',round(d['pcg_iteration']['us_per_iteration'],1),'us/it', d['config']['pcg_iters_per_step'])" || tail -3 gpurun_out/sweep/c${C}_u${U}_p${P}.err
    done
  done
done
