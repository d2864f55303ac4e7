cd $GRAFT_REPO_ROOT
timeout 300 python tools/gemm_timeline.py op 256 14336 4096 2 2>&1 | tail -12
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "gemm or mlp" 2>&1 | tail -2
