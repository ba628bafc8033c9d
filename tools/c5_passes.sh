# C5 at 384 / 1024: operator timings (bench_ops) and the per-pass DRAM throughput of one standalone normal
# operator + 2D FFT at 1024^2 x 32 under ncu (serialised, cold); summarise with tools/c5_summary.py
mkdir -p gpurun_out
timeout 600 python tools/bench_ops.py --ng 384,1024 --coils 12,32 > gpurun_out/c5_pk.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_pk_passes.csv python tools/normal_probe.py 1024 32 2 > /dev/null 2>&1
grep '"op"' gpurun_out/c5_pk.log | grep 1024
