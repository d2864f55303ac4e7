cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "attention or two_ctas" 2>&1 | tail -2
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
timeout 300 python tools/bench_attn.py attn_stages=3 2>&1 | tail -6
for t in "attn_stages=4" "attn_stages=3"; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --tuning $t > gpurun_out/s3k_bench_$t.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3k_bench_$t.json'));print('$t', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
done
