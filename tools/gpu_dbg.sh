cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=3 NS=128 timeout 300 python tools/dbg_batch.py 2>&1 | tail -4
CFG=3 NS=128 SBPCG_K1_G=2 timeout 300 python tools/dbg_batch.py 2>&1 | tail -4
CFG=3 NS=8 SBPCG_K1_G=1 timeout 300 python tools/dbg_batch.py 2>&1 | tail -4
CFG=4 NS=8 SBPCG_NO_PLANE=1 SBPCG_K1_G=1 timeout 300 python tools/dbg_batch.py 2>&1 | tail -4
CFG=4 NS=8 SBPCG_NO_PLANE=1 SBPCG_K1_G=2 timeout 300 python tools/dbg_batch.py 2>&1 | tail -4
