#!/bin/bash
# A/B of library variants on one box (under gpurun): tools/ab.sh NAME... where NAME is "base" (the in-tree
# libnlinv.so) or a file paper_1301_1215_b200/variants/NAME.so; bench.py twice per variant, interleaved.
mkdir -p gpurun_out
cp paper_1301_1215_b200/libnlinv.so /tmp/base.so
for rep in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_1301_1215_b200/libnlinv.so; else cp paper_1301_1215_b200/variants/$v.so paper_1301_1215_b200/libnlinv.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['latency_ms']['p50'], {k:round(1e3*v['ms']/v['launches'],2) for k,v in d['roofline']['kernels'].items() if k in ('col_k5_cg_k1','row_k4','col_psf','row_k2')})"
done; done
cp /tmp/base.so paper_1301_1215_b200/libnlinv.so
