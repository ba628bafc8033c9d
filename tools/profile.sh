#!/bin/bash
# Per-round ncu evidence (run under gpurun, one GPU). Writes into gpurun_out/.
set -x
mkdir -p gpurun_out
# 1) every launch of one frame with its device time (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_frame.py 1 > gpurun_out/launches.log 2>&1
# 2) full sets for the 7 kernels of one steady-state CG iteration (Newton step 0, CG iteration 2)
ncu --set full --clock-control none --import-source on \
    -k regex:'col_kernel|row_kernel|cg_update|rho_finish' -s 20 -c 7 \
    -o gpurun_out/prof_cg python tools/prof_frame.py 1 > gpurun_out/prof_cg.log 2>&1
ls -la gpurun_out
