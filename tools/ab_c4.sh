#!/bin/bash
# A/B of library variants on the C4 stream (32 coils, 384^2, 60 frames; tools/bench_stream.py) on one box:
# tools/ab_c4.sh NAME... with NAME "base" (in-tree libnlinv.so) or paper_1301_1215_b200/variants/NAME.so
cp paper_1301_1215_b200/libnlinv.so /tmp/base.so
for rep in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_1301_1215_b200/libnlinv.so; else cp paper_1301_1215_b200/variants/$v.so paper_1301_1215_b200/libnlinv.so; fi
  timeout 300 python tools/bench_stream.py --coils 32 --frames 60 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['device']['fps'], d['device']['latency_ms_p50'])"
done; done
cp /tmp/base.so paper_1301_1215_b200/libnlinv.so
