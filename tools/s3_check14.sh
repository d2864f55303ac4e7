cd $GRAFT_REPO_ROOT
for t in "partial_small_m=0" "partial_small_m=1"; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --tuning $t > gpurun_out/s3j_bench_$t.json 2> /dev/null
python -c "import json;d=json.load(open('gpurun_out/s3j_bench_$t.json'));print('$t', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
done
