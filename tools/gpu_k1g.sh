#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for G in 8 16 4; do
SBPCG_K1_G=$G timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_g.json 2>gpurun_out/b_g_err.log
python -c "import json;d=json.load(open('gpurun_out/b_g.json'));print('c2 G=$G',round(d['value']),'it/s',round(d['ms_per_step'],3),'ms K1',round(d['roofline']['kernel_avg_us'],2))"; tail -1 gpurun_out/b_g_err.log
done
timeout 300 python tools/prof_step.py --config 2 --eager > gpurun_out/plain2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_c2.csv python tools/prof_step.py --config 2 --eager > gpurun_out/ncu2.log 2>&1
python tools/launch_table.py gpurun_out/launches_c2.csv 2>/dev/null | head -8
