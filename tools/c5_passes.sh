mkdir -p gpurun_out
timeout 600 python tools/bench_ops.py --ng 384,1024 --coils 12,32 > gpurun_out/c5_pk.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c5_pk_passes.csv python tools/normal_probe.py 1024 32 2 > /dev/null 2>&1
grep '"op"' gpurun_out/c5_pk.log
