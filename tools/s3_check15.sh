cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_timeline.py op 16 4096 4096 1 2>&1 | tail -14
timeout 300 python tools/gemm_timeline.py op 32 6144 4096 0 2>&1 | tail -14
timeout 300 python tools/gemm_timeline.py op 32 4096 14336 1 2>&1 | tail -14
