cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --model qwen32b --steps 3 --warmup 3 --no-cpu > gpurun_out/s3_final_qwen32b.json 2> gpurun_out/s3_final_qwen32b.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s3_final_qwen32b.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], d['roofline']['frac'], d['decode_roofline_frac'] if 'decode_roofline_frac' in d else '', {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
