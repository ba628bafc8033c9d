#!/bin/bash
# A/B of the packed fp32x2 FFT arithmetic (default build) against the scalar build of the same code, on one
# box (run under gpurun): full GPU tests on the packed build, then bench.py twice per variant, interleaved.
# Build the scalar variant first (here): NLINV_DEFS=-DNLV_SCALAR_FP python -c "import __graft_entry__ as g; g.build()"
# && mkdir -p paper_1301_1215_b200/variants && cp paper_1301_1215_b200/libnlinv.so paper_1301_1215_b200/variants/scalarfp.so
# && python -c "import __graft_entry__ as g; g.build()"
mkdir -p gpurun_out
cp paper_1301_1215_b200/libnlinv.so /tmp/packed.so
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/packed_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/packed_pytest.log; tail -2 gpurun_out/packed_pytest.log
for rep in 1 2; do
for v in packed scalar; do
  if [ $v = packed ]; then cp /tmp/packed.so paper_1301_1215_b200/libnlinv.so; else cp paper_1301_1215_b200/variants/scalarfp.so paper_1301_1215_b200/libnlinv.so; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['latency_ms']['p50'], {k:round(1e3*v['ms']/v['launches'],2) for k,v in d['roofline']['kernels'].items() if k in ('col_k5_cg_k1','row_k4','col_psf','row_k2')})"
done; done
cp /tmp/packed.so paper_1301_1215_b200/libnlinv.so
