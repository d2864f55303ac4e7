# correctness of the fused variants, then engine-level timing
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_fullwidth.py tests/test_gpu_engine.py tests/test_gpu_ops.py -q -x -k "fullwidth_teacher_forced or fused_kernel_paths or small_m or mlp or attention" 2>&1 | tail -5
for t in "" "qkv_attn=1"; do
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu ${t:+--tuning $t} > gpurun_out/v.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('[$t]', round(d['value']), round(d['ms_per_decode_step'],3), d['clocks']['sm_mhz'], {k:round(v,3) for k,v in d['kernel_ms_per_decode_step'].items()})"
done
