set -x
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --tuning qkv_finish=1 > gpurun_out/r02_bench_qkvfinish.json 2>/dev/null
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --tuning fuse_mlp=0 > gpurun_out/r02_bench_nofuse.json 2>/dev/null
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python tools/ncu_steady.py 1500 > gpurun_out/ncu_steady.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:attn_bf16 -c 1 -o gpurun_out/r02_attn python tools/ncu_steady.py 1500 > gpurun_out/ncu_attn.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:mlp -c 1 -o gpurun_out/r02_mlp python tools/ncu_steady.py 1500 > gpurun_out/ncu_mlp.log 2>&1
for f in r02_bench_default r02_bench_qkvfinish r02_bench_nofuse; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], d['e2e']['value'] if d.get('e2e') else None, {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"; done
