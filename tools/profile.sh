#!/bin/bash
# Per-round ncu evidence (run under gpurun, one GPU). Writes into gpurun_out/.
mkdir -p gpurun_out
# 1) launch list of one C2 frame on the default path (fused cooperative passes, eager for ncu)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_default.csv python tools/prof_frame.py 1 > gpurun_out/launches_default.log 2>&1
# 2) full sets for one steady-state CG iteration (K2, K3, K4, fused K5+CG+K1) of Newton step 0
ncu --set full --clock-control none --import-source on \
    -k regex:'col_kernel|row_kernel' -s 13 -c 4 \
    -o gpurun_out/prof_iter python tools/prof_frame.py 1 > gpurun_out/prof_iter.log 2>&1
ls -la gpurun_out
