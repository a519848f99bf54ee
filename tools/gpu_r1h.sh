#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_3d.py tests/test_gpu_coil_mode.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -3
for C in 4 5 2; do
timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c$C.json 2> gpurun_out/bench_c${C}_err.log
python -c "import json;d=json.load(open('gpurun_out/bench_c$C.json'));r=d['roofline'];print('c$C',round(d['value']),'it/s',round(d['ms_per_step'],2),'ms',d['config']['pcg_iters_per_step'],'it/step K1',round(r['kernel_avg_us'],1),'us frac',round(r['frac'],3), d['config']['step_ms'])"; tail -2 gpurun_out/bench_c${C}_err.log
done
