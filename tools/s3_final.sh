cd $GRAFT_REPO_ROOT
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/s3_final_default.json 2> gpurun_out/s3_final_default.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s3_final_default.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks'], d['e2e']['value'], d['roofline']['frac'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
timeout 1200 python bench.py --full --no-cpu > gpurun_out/s3_final_full.json 2> gpurun_out/s3_final_full.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s3_final_full.json'));print({k:d[k] for k in d if k in ('value','ms_per_decode_step','bubble','decode_roofline_frac','since_start_steps','clocks')})"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s3_final_ref.json 2>/dev/null; echo ref rc=$?; tail -c 400 gpurun_out/s3_final_ref.json
