cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ops.py -q -x -k "sample or trunc" 2>&1 | tail -2
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3h_launches.csv python tools/ncu_steady.py 1500 > gpurun_out/s3h_ncu_steady.log 2>&1; echo ncu rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/s3h_bench.json 2> gpurun_out/s3h_bench.err
python -c "import json;d=json.load(open('gpurun_out/s3h_bench.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
