cd $GRAFT_REPO_ROOT
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s3_final2_bench.json 2> gpurun_out/s3_final2_bench.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s3_final2_bench.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['cpu_baseline']['value'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
