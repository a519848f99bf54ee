#!/bin/bash
# ncu metric pass (not --set full): DRAM bytes, FMA-pipe busy, issue-active and warps-active of
# the dominant kernel of every config (the FP32-issue co-limit of SURVEY 8(d)); summarised by
# tools/pipes_summary.py into profiles/ncu_pipes.json and profiles/ncu_traffic.json.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pipes
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.sum,smsp__inst_executed.sum
for spec in "2 k_persist 0" "3 k1_matvec<\(int\)256, \(int\)8, \(int\)1> 2" "4 kp_plane<\(int\)256, \(int\)128, \(int\)16, \(int\)1> 2" "5 kp_plane<\(int\)192, \(int\)192, \(int\)8, \(int\)1> 1"; do
  set -- $spec
  C=$1; S=${@: -1}; K="${*:2:$#-2}"
  timeout 600 python tools/prof_step.py --config $C --eager --steps 1 --warmup 1 > gpurun_out/pipes/plain$C.log 2>&1 || { echo "plain $C failed"; continue; }
  timeout 900 ncu --metrics $M --clock-control none --kernel-name-base demangled -k "regex:$K" -s $S -c 3 --profile-from-start off \
    --csv --log-file gpurun_out/pipes/c$C.csv python tools/prof_step.py --config $C --eager --steps 1 --warmup 1 > gpurun_out/pipes/ncu$C.log 2>&1
  echo "config $C: $(grep -c gpu__time_duration gpurun_out/pipes/c$C.csv) rows"
done
