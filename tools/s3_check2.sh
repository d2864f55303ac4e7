cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x 2>&1 | tail -4
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3b_timeline.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3b_bench.json 2> gpurun_out/s3b_bench.err
python -c "import json;d=json.load(open('gpurun_out/s3b_bench.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --tuning stream_n=0 > gpurun_out/s3b_bench_sn0.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3b_bench_sn0.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
