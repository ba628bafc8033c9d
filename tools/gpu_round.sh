#!/bin/bash
# One gpurun round trip: probe, GPU tests, bench, sanitizers (tag = $1). Logs in gpurun_out/.
TAG=${1:-r2}
mkdir -p gpurun_out
bash tools/probe.sh > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
bash tools/sanitize.sh > /dev/null 2>&1
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/sanitize_summary.txt; tail -1 gpurun_out/${TAG}_bench.log | head -c 1500
