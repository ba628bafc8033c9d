#!/bin/bash
# warm-cache DRAM vs L2 traffic of one steady-state CG iteration (no cache flush between kernels)
mkdir -p gpurun_out
ncu --cache-control none --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.per_cycle_active \
    -k regex:'col_kernel|row_kernel|cg_update|rho_finish' -s 20 -c 14 --csv --log-file gpurun_out/warm.csv \
    python tools/prof_frame.py 1 > gpurun_out/warm.log 2>&1
