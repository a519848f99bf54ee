#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
TAG=U1 CFG=2 timeout 300 python tools/step_times.py
TAG=U1 CFG=2 timeout 300 python tools/step_times.py
TAG=U2 SBPCG_UNROLL=2 CFG=2 timeout 300 python tools/step_times.py
TAG=U3 SBPCG_UNROLL=3 CFG=2 timeout 300 python tools/step_times.py
TAG=U1 CFG=3 N=6 timeout 300 python tools/step_times.py
TAG=U2 SBPCG_UNROLL=2 CFG=3 N=6 timeout 300 python tools/step_times.py
