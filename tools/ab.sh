#!/bin/bash
# A/B of an env switch on the C2 bench (tag, VAR=VALUE): parity subset first
TAG=${1:-ab}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
for i in 1 2; do
  for v in "" "$@"; do
    env $v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_b.log 2>&1
    echo "[$v] $(tail -1 gpurun_out/${TAG}_b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fps',d['value'],'e2e',d['e2e']['value'], {k:(v['ms'],v['launches']) for k,v in list(d['roofline']['kernels'].items())[:5]})")"
  done
done
