cd $GRAFT_REPO_ROOT
BENCH_M=256,192,128,96,64,32,16 timeout 600 python tools/bench_ops.py 2>&1 | grep -v "^attn" | tail -45
