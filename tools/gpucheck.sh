#!/bin/bash
# One gpurun round trip: GPU parity tests + bench (default args). Logs land in gpurun_out/.
mkdir -p gpurun_out
tag=${1:-check}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 400 python bench.py ${BENCH_ARGS} > gpurun_out/${tag}_bench.log 2>&1
tail -2 gpurun_out/${tag}_pytest.log
tail -1 gpurun_out/${tag}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps',d['value'],'e2e',d['e2e']['value'],{k:(v['ms'],v['launches']) for k,v in d['roofline']['kernels'].items()})"
