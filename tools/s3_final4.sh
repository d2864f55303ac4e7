cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=clocks.max.sm --format=csv
timeout 1200 python bench.py --full --no-cpu > gpurun_out/s3_final4_full.json 2> gpurun_out/s3_final4_full.err; echo rc=$?
python -c "import json;d=json.load(open('gpurun_out/s3_final4_full.json'));print(round(d['value']), round(d['ms_per_decode_step'],3), d['decode_steps'], d['clocks'], d['decode_roofline_frac']['value'], d['bubble_ratio'])"
