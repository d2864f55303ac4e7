cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_compact.py -q -x 2>&1 | tail -2
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3i_timeline.txt 2>&1; sed -n '/gate_up/,/down/p' gpurun_out/s3i_timeline.txt
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3i_bench.json 2> gpurun_out/s3i_bench.err
python -c "import json;d=json.load(open('gpurun_out/s3i_bench.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
