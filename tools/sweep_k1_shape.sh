#!/bin/bash
# K1 wave quantisation and tile width on config 3: per-problem PCG iteration time at batch sizes
# that fill whole waves of 444 resident CTAs (3 per SM; 32 tiles per problem) or not, and W = 4.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/sweep
run() {  # tag, env, slices
  env $2 timeout 600 python bench.py --config 3 --slices $3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra \
    > gpurun_out/sweep/k1_$1.json 2> gpurun_out/sweep/k1_$1.err
  python -c "import json;d=json.load(open('gpurun_out/sweep/k1_$1.json'));p=d['pcg_iteration'];r=d['roofline'];print('$1 slices=$3',round(p['us_per_iteration'],1),'us/it',round(p['us_per_iteration']/$3,3),'us/it/problem', 'K1', round(r['kernel_avg_us'],1),'us', round(r['frac'],3))" || tail -3 gpurun_out/sweep/k1_$1.err
}
run w8_s111 "SBPCG_K1_W=8" 111
run w8_s120 "SBPCG_K1_W=8" 120
run w8_s128 "SBPCG_K1_W=8" 128
run w4_s128 "SBPCG_K1_W=4" 128
run w4_s111 "SBPCG_K1_W=4" 111
