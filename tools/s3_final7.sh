cd $GRAFT_REPO_ROOT
T0=$(date +%s); timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_final7_ref.json 2> gpurun_out/s3_final7_ref.err; echo ref rc=$?; tail -1 gpurun_out/s3_final7_ref.err
python -c "import json;d=json.load(open('gpurun_out/s3_final7_ref.json'));print({k:d[k] for k in ('impl','value','unit','ms_per_step','steps','warmup')})"
T1=$(date +%s); echo ref wall $((T1-T0)) s; timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/s3_final7_ours.json 2> gpurun_out/s3_final7_ours.err; echo ours rc=$?; tail -1 gpurun_out/s3_final7_ours.err
python -c "import json;d=json.load(open('gpurun_out/s3_final7_ours.json'));print(round(d['value']), d['clocks'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['traffic'], d['gpu_launches'], d['cpu_baseline']['value'])"
echo ours wall $(( $(date +%s) - T1 )) s
