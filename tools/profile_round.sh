#!/bin/bash
# Round evidence beyond tools/profile.sh (one GPU, under gpurun): a graph-mode C2 frame under ncu, the
# cluster-fused pass's launch list, the C5 operator sweep, f4 micro-benchmarks, C4 / C1 streams.
# Outputs in gpurun_out/ (TAG prefix); summarise into profiles/.
TAG=${1:-r02}
mkdir -p gpurun_out
# graph-mode C2 frame: ncu profiles the whole CUDA graph of a frame as one unit (frame 0 cold start, 1-2 warm)
ncu --graph-profiling graph --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_graph_frame.csv \
    python tools/prof_frame_graph.py 3 > gpurun_out/${TAG}_graph_frame.log 2>&1
# the cluster-fused K2-K3-K4 pass (opt-in) next to the three passes it replaces, cold cache
NLINV_K234=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_launches_k234.csv python tools/prof_frame.py 1 > /dev/null 2>&1
timeout 900 python tools/bench_ops.py > gpurun_out/${TAG}_c5.log 2>&1
timeout 300 python tools/bench_micro.py > gpurun_out/${TAG}_micro.json 2>&1
timeout 600 python tools/bench_stream.py --coils 32 --frames 200 > gpurun_out/${TAG}_c4.log 2>&1
timeout 600 python tools/bench_stream.py --coils 8 --ng 32 --spokes 8 --turns 1 --newton 3 --frames 200 > gpurun_out/${TAG}_c1.log 2>&1
ls -la gpurun_out | tail -20
