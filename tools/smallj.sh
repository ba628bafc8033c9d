# frame time vs coils per GPU (the per-rank load of coil-sharded runs) for library variants:
# tools/smallj.sh base|VARIANT... (VARIANT = paper_1301_1215_b200/variants/VARIANT.so)
cp paper_1301_1215_b200/libnlinv.so /tmp/base.so
for v in "$@"; do
  if [ $v = base ]; then cp /tmp/base.so paper_1301_1215_b200/libnlinv.so; else cp paper_1301_1215_b200/variants/$v.so paper_1301_1215_b200/libnlinv.so; fi
  for J in 1 2 3 4 6 12; do timeout 300 python tools/bench_stream.py --coils $J --frames 60 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v J=$J', d['device']['fps'], d['device']['latency_ms_p50'])"; done
done
cp /tmp/base.so paper_1301_1215_b200/libnlinv.so
