#!/bin/bash
# Per-round ncu evidence (run under gpurun, one GPU). Writes into gpurun_out/; summarise with
# python tools/ncu_summary.py (writes profiles/).
mkdir -p gpurun_out
# 1) launch list of one C2 frame on the default path (eager launches for ncu), cold cache per kernel
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cold.csv python tools/prof_frame.py 1 > gpurun_out/launches_cold.log 2>&1
# 2) the same with warm caches (no flush between kernels): the L2-resident reality of a frame
ncu --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct \
    --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/prof_frame.py 1 > gpurun_out/launches_warm.log 2>&1
# 3) full sets for one steady-state CG iteration (K2, K3, K4, fused K5+CG+K1) of Newton step 0
ncu --set full --clock-control none --import-source on \
    -k regex:'col_kernel|row_kernel|k5cg' -s 13 -c 4 \
    -o gpurun_out/prof_iter python tools/prof_frame.py 1 > gpurun_out/prof_iter.log 2>&1
ls -la gpurun_out
