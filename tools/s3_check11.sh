cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_timeline.py op 256 14336 4096 2 2>&1 | tail -12
