cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_ops.py -q -x -k "gemm or mlp or rmsnorm or norm" 2>&1 | tail -2
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3l_timelineA.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3l_benchA.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3l_benchA.json'));print('A(regcap)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
cp tools/varB/gemm_pair.cuh paper_2603_23414_b200/csrc/gemm_pair.cuh; cp tools/varB/layers.cu paper_2603_23414_b200/csrc/layers.cu
python -c "from paper_2603_23414_b200 import build; build.build(force=True)" 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3l_benchB.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3l_benchB.json'));print('B(orig)', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
