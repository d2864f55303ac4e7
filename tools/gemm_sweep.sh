#!/bin/bash
# GEMM config sweep at M=256 (srl_tuning overrides of the launcher's H / stage choices)
for cfg in "1 0 0" "1 0 1" "1 6 3" "1 4 4" "2 0 0" "2 4 1" "2 3 2" "2 2 3"; do
  set -- $cfg
  echo "== H=$1 stages=$2 xstages=$3"
  BENCH_TUNING="gemm_h=$1,gemm_stages=$2,gemm_xstages=$3" BENCH_M=256 timeout 120 python tools/bench_ops.py 2>&1 | grep "M256" | python -c "
import sys, json
for l in sys.stdin:
    n, d = l.split(' ', 1); d = json.loads(d); print(f'  {n:14s} {d[\"us\"]:8.2f} us {d[\"weight_GBs\"]:7.0f} GB/s')"
done
