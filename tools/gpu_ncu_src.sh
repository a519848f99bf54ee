#!/bin/bash
# ncu --set full with source-level (SASS) stall sampling of the K1P PCG launch, configs 4 and 5.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/src
for spec in "4 3" "5 2"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:kp_plane<.*\(int\)1>" -s $2 -c 1 --profile-from-start off \
    -o gpurun_out/src/full_c$1 -f python tools/prof_step.py --config $1 --eager --steps 1 --warmup 1 > gpurun_out/src/ncuf$1.log 2>&1
  ncu -i gpurun_out/src/full_c$1.ncu-rep --page source --csv --print-source sass > gpurun_out/src/src_c$1.csv 2>/dev/null
  ncu -i gpurun_out/src/full_c$1.ncu-rep --page details --csv > gpurun_out/src/det_c$1.csv 2>/dev/null
  rm -f gpurun_out/src/full_c$1.ncu-rep
  tail -1 gpurun_out/src/ncuf$1.log; ls -la gpurun_out/src/src_c$1.csv
done
