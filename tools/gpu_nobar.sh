#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for C in 4 5; do for E in 0 1; do
SBPCG_DBG_NOBAR=$E TAG="nobar=$E" CFG=$C timeout 300 python tools/time_applyA.py 2>&1 | tail -1
done; done
