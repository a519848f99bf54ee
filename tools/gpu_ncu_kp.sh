#!/bin/bash
# ncu --set full of the plane matvec (config $CFG) + raw/source pages
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CFG=${CFG:-5}
K=${K:-kp_plane}
timeout 300 python tools/prof_step.py --config $CFG --eager --steps 1 --warmup 0 > gpurun_out/plainkp.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s ${SKIP:-3} -c 1 --profile-from-start off \
  -o gpurun_out/kp_c$CFG -f python tools/prof_step.py --config $CFG --eager --steps 1 --warmup 0 > gpurun_out/ncukp.log 2>&1
tail -3 gpurun_out/ncukp.log
ncu -i gpurun_out/kp_c$CFG.ncu-rep --page raw --csv > gpurun_out/kp_c${CFG}_raw.csv 2>/dev/null
ncu -i gpurun_out/kp_c$CFG.ncu-rep --page source --csv > gpurun_out/kp_c${CFG}_src.csv 2>/dev/null
ncu -i gpurun_out/kp_c$CFG.ncu-rep --page details --csv > gpurun_out/kp_c${CFG}_details.csv 2>/dev/null
ls -la gpurun_out/kp_c$CFG*
