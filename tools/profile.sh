#!/bin/bash
# Per-round ncu evidence (run under gpurun, one GPU). Writes into gpurun_out/.
mkdir -p gpurun_out
# 1) launch list of one C2 frame, default path (persistent frame kernel)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_frame.csv python tools/prof_frame.py 1 > gpurun_out/launches_frame.log 2>&1
# 2) launch list of one C2 frame, multi-kernel path (per-pass breakdown)
NLINV_NO_FRAME=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_multi.csv python tools/prof_frame.py 1 > gpurun_out/launches_multi.log 2>&1
# 3) full set on the frame kernel (one launch = one frame)
ncu --set full --clock-control none --import-source on -k regex:frame_kernel -c 1 \
    -o gpurun_out/prof_frame python tools/prof_frame.py 1 > gpurun_out/prof_frame.log 2>&1
# 4) full set on the 7 kernels of one steady-state CG iteration of the multi-kernel path
NLINV_NO_FRAME=1 ncu --set full --clock-control none --import-source on \
    -k regex:'col_kernel|row_kernel|cg_update' -s 18 -c 6 \
    -o gpurun_out/prof_cg python tools/prof_frame.py 1 > gpurun_out/prof_cg.log 2>&1
ls -la gpurun_out
