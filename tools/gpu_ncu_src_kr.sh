#!/bin/bash
# ncu source-level stall sampling of KR (config 2) and K1 (config 3, PCG mode).
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/src
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_persist" -c 1 --profile-from-start off \
  -o gpurun_out/src/full_c2 -f python tools/prof_step.py --config 2 --eager --steps 1 --warmup 1 > gpurun_out/src/ncuf2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k1_matvec<.*\(int\)1>" -s 3 -c 1 --profile-from-start off \
  -o gpurun_out/src/full_c3 -f python tools/prof_step.py --config 3 --eager --steps 1 --warmup 1 > gpurun_out/src/ncuf3.log 2>&1
for C in 2 3; do
  ncu -i gpurun_out/src/full_c$C.ncu-rep --page source --csv --print-source sass > gpurun_out/src/src_c$C.csv 2>/dev/null
  rm -f gpurun_out/src/full_c$C.ncu-rep
  tail -1 gpurun_out/src/ncuf$C.log; ls -la gpurun_out/src/src_c$C.csv
done
