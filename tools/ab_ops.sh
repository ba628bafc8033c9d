#!/bin/bash
# A/B of library variants on the C5 operator sweep (tools/bench_ops.py) on one box (under gpurun):
# tools/ab_ops.sh NGS COILS NAME... with NAME "base" (in-tree libnlinv.so) or paper_1301_1215_b200/variants/NAME.so
NGS=$1; COILS=$2; shift 2
cp paper_1301_1215_b200/libnlinv.so /tmp/base.so
for rep in 1 2; do
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_1301_1215_b200/libnlinv.so; else cp paper_1301_1215_b200/variants/$v.so paper_1301_1215_b200/libnlinv.so; fi
  timeout 300 python tools/bench_ops.py --ng $NGS --coils $COILS --reps 30 2>&1 | grep '"op"' | sed "s/^/$v /"
done; done
cp /tmp/base.so paper_1301_1215_b200/libnlinv.so
