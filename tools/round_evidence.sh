#!/bin/bash
# round evidence on the final code (TAG = $1): GPU tests, bench, sanitizers, ncu launch lists, C4 / C1 streams, C5 sweep, small-J
TAG=${1:-r02e}
mkdir -p gpurun_out
bash tools/gpu_round.sh $TAG > gpurun_out/${TAG}_round.txt 2>&1
bash tools/profile.sh > /dev/null 2>&1
timeout 600 python tools/bench_stream.py --coils 32 --frames 200 > gpurun_out/${TAG}_c4.log 2>&1
timeout 600 python tools/bench_stream.py --coils 8 --ng 32 --spokes 8 --turns 1 --newton 3 --frames 200 > gpurun_out/${TAG}_c1.log 2>&1
timeout 900 python tools/bench_ops.py > gpurun_out/${TAG}_c5.log 2>&1
bash tools/smallj.sh base > gpurun_out/${TAG}_smallj.txt 2>&1
cat gpurun_out/${TAG}_round.txt; tail -1 gpurun_out/${TAG}_c4.log | head -c 600; echo; cat gpurun_out/${TAG}_smallj.txt
