cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py tests/test_gpu_engine.py -q -x -k "attention or parity or two_epochs or qkv" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullwidth.py -q -x -k "llama8b or long_context" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3o_benchA.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3o_benchA.json'));print('A(pre)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
cp tools/varB/attention.cu paper_2603_23414_b200/csrc/attention.cu
python -c "from paper_2603_23414_b200 import build; build.build(force=True)" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3o_benchB.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3o_benchB.json'));print('B(orig)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
