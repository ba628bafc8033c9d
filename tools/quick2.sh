#!/bin/bash
# multi-rank tests + parity subset + short bench (tag = $1)
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/${TAG}_mr.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_mr.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_frames.py -m gpu -x -q -k "not c2_warm and not 384-12-15-5-7" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1
tail -15 gpurun_out/${TAG}_mr.log
tail -3 gpurun_out/${TAG}_pytest.log
tail -1 gpurun_out/${TAG}_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps',d['value'],'e2e',d['e2e']['value'],d['latency_ms'])"
