# N1 / N4 whole-path measurements on the cfg2 engine (20 early-update rounds each) + sanitizers
cd $GRAFT_REPO_ROOT
run() { name=$1; shift; timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu "$@" > gpurun_out/r02_bench_$name.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/r02_bench_$name.json'));print('$name', round(d['value']), 'useful', round(d['useful_tokens_per_s']), round(d['ms_per_decode_step'],3), d['decode_steps'], d['clocks']['sm_mhz'], 'prefill_ms/step', round(d['kernel_ms_per_decode_step'].get('prefill',0),3), 'bubble', round(d['bubble_ratio']['window_abstract'],3))"; }
run K1_keepkv --K 1
run K1_reprefill --K 1 --resume reprefill
run K1_reprefill_C4096 --K 1 --resume reprefill --prefill-budget 4096
run G8 --G 8
run G8_share --G 8 --share-prefix
timeout 600 compute-sanitizer --tool memcheck --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -3 gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitizer_racecheck.log
