#!/bin/bash
set -u
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 | tee gpurun_out/r02h_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee -a gpurun_out/r02h_gpu_tests.txt
timeout 900 python bench.py > gpurun_out/r02h_bench_default.json 2> gpurun_out/bench_default_err.log; tail -c 1500 gpurun_out/r02h_bench_default.json; tail -2 gpurun_out/bench_default_err.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02h_bench_ref.json 2> gpurun_out/bench_ref_err.log; tail -c 800 gpurun_out/r02h_bench_ref.json
