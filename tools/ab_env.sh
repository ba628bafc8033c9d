#!/bin/bash
# A/B of environment switches on one box (under gpurun): tools/ab_env.sh "VAR=VAL ..." ... ("-" = none);
# bench.py twice per setting, interleaved
for rep in 1 2; do
for v in "$@"; do
  e=""; [ "$v" != "-" ] && e="$v"
  env $e timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['latency_ms']['p50'], {k:round(1e3*v['ms']/v['launches'],2) for k,v in d['roofline']['kernels'].items() if k in ('col_k5_cg_k1','row_k4','col_psf','row_k2')})"
done; done
