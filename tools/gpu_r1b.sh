#!/bin/bash
# round-1 session-2 GPU cycle: config-4 bench + launch list; ncu --set full of K1 (configs 2, 3)
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4_err.log; tail -c 2500 gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4_err.log
timeout 300 python tools/prof_step.py --config 4 --eager > gpurun_out/plain4.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_c4.csv python tools/prof_step.py --config 4 --eager > gpurun_out/ncu4.log 2>&1
python tools/launch_table.py gpurun_out/launches_c4.csv 2>/dev/null | head -16
for C in 2 3; do
timeout 300 python tools/prof_step.py --config $C --eager > gpurun_out/plain$C.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k1_matvec -s 20 -c 2 --profile-from-start off \
  -o gpurun_out/k1_c$C -f python tools/prof_step.py --config $C --eager > gpurun_out/ncufull$C.log 2>&1
ncu -i gpurun_out/k1_c$C.ncu-rep --page raw --csv > gpurun_out/k1_c${C}_raw.csv 2>/dev/null
python tools/ncu_traffic.py gpurun_out/k1_c${C}_raw.csv $C
done
