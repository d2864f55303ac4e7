cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "gemm" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fullwidth.py -q -x -k "norm_prologue or llama8b" 2>&1 | tail -3
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3d_timeline.txt 2>&1; tail -1 gpurun_out/s3d_timeline.txt
for t in "norm_pro=1,pair_h2=1" "norm_pro=0,pair_h2=1" "norm_pro=1,pair_h2=0" "norm_pro=0,pair_h2=0"; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --tuning $t > gpurun_out/s3d_bench_$t.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3d_bench_$t.json'));print('$t', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
done
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
