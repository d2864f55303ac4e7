cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,power.limit --format=csv
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3_timeline.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3_bench.json 2> gpurun_out/s3_bench.err
tail -c 3000 gpurun_out/s3_bench.json
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
