#!/bin/bash
# ncu full set of the cluster-fused K2-K3-K4 kernel and the k5cg pass of one CG iteration (C2)
mkdir -p gpurun_out
python tools/cluster_probe.py > gpurun_out/cluster_probe.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:'k234|k5cg' -s 4 -c 2 \
    -o gpurun_out/prof_k234 python tools/prof_frame.py 1 > gpurun_out/prof_k234.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_k234.csv \
    python tools/prof_frame.py 1 > /dev/null 2>&1
cat gpurun_out/cluster_probe.txt
