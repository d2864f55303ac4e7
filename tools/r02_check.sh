cd $GRAFT_REPO_ROOT
timeout 300 ./tools/stream_bench.bin 2>&1 | sort -t' ' -k7 -n | tail -8
timeout 300 python tools/bench_attn.py 2>&1 | tail -6
timeout 300 python tools/bench_attn.py attn_stages=6 2>&1 | tail -6
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --error-exitcode 9 python __graft_entry__.py smoke > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/sanitizer_racecheck.log
