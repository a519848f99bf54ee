#!/bin/bash
# Profiling pass: eager launch lists (configs 2-5) and ncu --set full of the
# dominant kernel per config (the persistent kernel KR for 2, K1 for 3, K1P for 4/5), raw pages
# exported for the summaries (tools/summarize_profiles.py).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/prof
for C in 2 3 4 5; do
  timeout 400 python tools/prof_step.py --config $C --eager --steps 1 --warmup 1 > gpurun_out/prof/plain$C.log 2>&1 || { echo "plain $C failed"; tail -3 gpurun_out/prof/plain$C.log; continue; }
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/prof/launches_c$C.csv python tools/prof_step.py --config $C --eager --steps 1 --warmup 1 > gpurun_out/prof/ncul$C.log 2>&1
  echo "== config $C"; python tools/launch_table.py gpurun_out/prof/launches_c$C.csv 2>/dev/null | head -14
done
# the PCG-mode instance (template MODE 1) of the dominant kernel
for spec in "2 k_persist 0" "3 k1_matvec 3" "4 kp_plane 3" "5 kp_plane 2"; do
  set -- $spec
  K="regex:$2<.*\(int\)1>"
  [ "$2" = k_persist ] && K="regex:k_persist"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "$K" -s $3 -c 1 --profile-from-start off \
    -o gpurun_out/prof/full_c$1 -f python tools/prof_step.py --config $1 --eager --steps 1 --warmup 1 > gpurun_out/prof/ncuf$1.log 2>&1
  ncu -i gpurun_out/prof/full_c$1.ncu-rep --page raw --csv > gpurun_out/prof/full_c$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/full_c$1.ncu-rep --page details --csv > gpurun_out/prof/full_c$1_details.csv 2>/dev/null
  ncu -i gpurun_out/prof/full_c$1.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/full_c${1}_src.csv 2>/dev/null
  rm -f gpurun_out/prof/full_c$1.ncu-rep
  tail -1 gpurun_out/prof/ncuf$1.log
done
ls gpurun_out/prof | head -40
