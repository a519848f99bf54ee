#!/bin/bash
# Results pass for DESIGN.md §7: smoke, the default bench line (config 2, full contract), the
# other configs' bench lines (with e2e), and the reference (oracle) arm.
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/results
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/results/c2.json 2> gpurun_out/results/c2.err; tail -c 3000 gpurun_out/results/c2.json
for C in 3 4 5; do
  S=5; [ $C = 5 ] && S=3
  timeout 900 python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/results/c$C.json 2> gpurun_out/results/c$C.err
  python -c "import json;d=json.load(open('gpurun_out/results/c$C.json'));print('c$C',round(d['value'],1),d['unit'],'e2e',round(d['e2e']['value'],1),'step',round(d['ms_per_step'],2),'ms frac',d['roofline']['frac'],'iter',d['pcg_iteration'])" || tail -3 gpurun_out/results/c$C.err
done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/results/ref.json 2> gpurun_out/results/ref.err; tail -c 1500 gpurun_out/results/ref.json
