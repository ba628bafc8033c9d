#!/bin/bash
mkdir -p gpurun_out
timeout 120 compute-sanitizer --tool memcheck --print-limit 2 python tools/dbg_ops.py 48 3 2>&1 | grep -E "ok|Access at|Invalid|ERROR SUMMARY" | head -12
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -m gpu -x -q > gpurun_out/par.log 2>&1; echo "rc=$?" >> gpurun_out/par.log; tail -3 gpurun_out/par.log
