cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3e_bench.json 2> gpurun_out/s3e_bench.err
python -c "import json;d=json.load(open('gpurun_out/s3e_bench.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], d['e2e']['value'], d['roofline']['frac'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
timeout 300 python tools/gemm_timeline.py engine 4 > gpurun_out/s3e_timeline.txt 2>&1; tail -1 gpurun_out/s3e_timeline.txt
timeout 300 python tools/bench_attn.py > gpurun_out/s3e_attn.txt 2>&1; cat gpurun_out/s3e_attn.txt
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3e_launches.csv python tools/ncu_steady.py 1500 > gpurun_out/s3e_ncu_steady.log 2>&1; echo ncu rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_pair_kernel -s 2 -c 1 -o gpurun_out/s3e_gateup python tools/ncu_steady.py 1500 > gpurun_out/s3e_ncu_gu.log 2>&1; echo ncu2 rc=$?
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
