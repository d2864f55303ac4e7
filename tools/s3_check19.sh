cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "attention or two_ctas" 2>&1 | tail -2
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3n_benchA.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3n_benchA.json'));print('A(new)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
cp tools/varB/attention.cu paper_2603_23414_b200/csrc/attention.cu
python -c "from paper_2603_23414_b200 import build; build.build(force=True)" 2>&1 | tail -2
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3n_benchB.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3n_benchB.json'));print('B(orig)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
