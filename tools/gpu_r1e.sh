#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for C in 2 3 4; do
timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$C.json 2> gpurun_out/bench_c${C}_err.log
python -c "import json;d=json.load(open('gpurun_out/bench_c$C.json'));r=d['roofline'];print('c$C',round(d['value']),'it/s',round(d['ms_per_step'],2),'ms',d['config']['pcg_iters_per_step'],'it/step K1',round(r['kernel_avg_us'],1),'us frac',round(r['frac'],3))"; tail -2 gpurun_out/bench_c${C}_err.log
done
timeout 300 python tools/prof_step.py --config 2 --eager > gpurun_out/plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_c2.csv python tools/prof_step.py --config 2 --eager > gpurun_out/ncu2.log 2>&1
python tools/launch_table.py gpurun_out/launches_c2.csv 2>/dev/null | head -12
CFG=5 bash tools/gpu_ncu_kp.sh
